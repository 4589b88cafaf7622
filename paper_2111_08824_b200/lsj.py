"""Learned sort-join on the GPU (reference lsj.py:1-405).

Per relation (``prepare_model`` + ``sort_relation``):

* smpl: a stratified sample of ``sample_rate`` of the keys, sorted on device;
  the reference's two-level linear RMI fitted on it (K10, models.py:57-110,
  fanout min(1000, samples // 8) as lsj.py:127-129); equi-depth bins over
  the model's predicted positions, cut at equally spaced sample ranks
  (bin(key) = table[pos(key)], monotone in the key).
* part: K6/K7 shared-memory-privatised histogram + scatter into the bins.
* sort: K8 model-placed per-bucket sort in shared memory (oversized buckets
  re-partitioned by the model at finer resolution).

Then ``chunked_join`` (K9) walks sorted S in tiles; each tile's R window is
found through R's model and bucket bounds.  The result is the checksum
(count, sum, xor) of R.payload + S.payload over all equal-key pairs (pairs
on request).  The reference's bucket scale P = ``effective_fanout`` is kept
for the API, the ModelMismatch guard and the sort counters
(comparator_count / partitions_sorted are computed exactly from the bucket
sizes at scale P, tests/test_lsj.py:27-32).
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .data import RecordRelation, Relation
from .models import RecursiveModelIndex
from .results import JoinResult, PhaseBreakdown, SortStats
from .util import exclusive_offsets, to_device_u64, unsigned_order

BUCKET_TARGET = 8192  # mean tuples per sort unit (the shared-memory sort holds <= 12288)
# coarse bins of the grid-wide partition (open write lines stay in L2); LJ_LSJ_MAX_BINS: tuning experiments
MAX_BINS = min(2048, max(1, int(os.environ.get("LJ_LSJ_MAX_BINS", "2048"))))


class ModelMismatchError(ValueError):
    """A sorted relation was joined under a model/scale it was not built with."""


@dataclass(frozen=True)
class LsjConfig:
    """lsj.py:30-68."""

    workers: int = 1
    sample_rate: float = 0.01
    fanout: int = 10000
    swwc: bool = True
    swwc_buf_len: int = 64
    overalloc: float = 0.02
    model_fanout: int | None = None
    seed: int = 0x1D5EED

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if not 0.0 < self.sample_rate <= 1.0:
            raise ValueError("sample_rate must be in (0, 1]")
        if self.fanout < self.workers:
            raise ValueError("fanout must be >= workers")
        if self.swwc_buf_len < 1:
            raise ValueError("swwc_buf_len must be >= 1")
        if self.overalloc < 0.0:
            raise ValueError("overalloc must be >= 0")

    def effective_fanout(self) -> int:
        """Sort-phase partition count, a multiple of workers (lsj.py:53-56)."""
        return -(-self.fanout // self.workers) * self.workers

    def as_dict(self) -> dict:
        return {"workers": self.workers, "sample_rate": self.sample_rate, "fanout": self.fanout,
                "swwc": self.swwc, "swwc_buf_len": self.swwc_buf_len, "overalloc": self.overalloc,
                "model_fanout": self.model_fanout, "seed": self.seed}


class LsjModel:
    """An RMI plus bins over its predicted positions (LjLsjModel)."""

    def __init__(self, rmi: RecursiveModelIndex, pb: torch.Tensor, table: torch.Tensor,
                 sample: torch.Tensor | None = None):
        self.rmi = rmi
        self.pb = pb
        self.table = table
        self.nbins = pb.numel() - 1
        self.sample = sample

    @property
    def tag(self):
        return self.rmi.tag

    def c_struct(self) -> _lib.LjLsjModel:
        ns = self.sample.numel() if self.sample is not None else 0
        return _lib.LjLsjModel(self.rmi.c_struct(), self.nbins, _lib.ptr(self.pb), _lib.ptr(self.table),
                               _lib.ptr(self.sample), ns)

    @classmethod
    def uniform(cls, rmi: RecursiveModelIndex, nbins: int) -> "LsjModel":
        """Bins = the reference's partition_index buckets at scale nbins
        (pb[j] = ceil(j * n / nbins))."""
        tl = rmi.trained_len
        j = np.arange(nbins + 1, dtype=np.int64)
        pb = torch.from_numpy(-((-j * tl) // nbins)).to(rmi.leaves.device)
        table = torch.empty(tl, dtype=torch.int32, device=pb.device)
        _lib.check(_lib.lib().lj_lsj_bins_from_bounds(_lib.ptr(pb), nbins, tl, _lib.ptr(table),
                                                      _lib.stream_ptr()), "lsj_bins")
        return cls(rmi, pb, table)

    @classmethod
    def from_sample(cls, rmi: RecursiveModelIndex, sample_sorted: torch.Tensor, nbins: int) -> "LsjModel":
        """Equi-depth bins cut at equally spaced sample ranks."""
        lib = _lib.lib()
        dev = sample_sorted.device
        pb = torch.empty(nbins + 1, dtype=torch.int64, device=dev)
        table = torch.empty(rmi.trained_len, dtype=torch.int32, device=dev)
        ws = _lib.workspace(lib.lj_lsj_bins_workspace_bytes(sample_sorted.numel()), dev)
        c = rmi.c_struct()
        _lib.check(lib.lj_lsj_bins(ctypes.byref(c), _lib.ptr(sample_sorted), sample_sorted.numel(), nbins,
                                   _lib.ptr(pb), _lib.ptr(table), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
                   "lsj_bins")
        return cls(rmi, pb, table, sample_sorted)


def default_bins(n: int) -> int:
    return max(1, min(MAX_BINS, math.ceil(n / BUCKET_TARGET)))


@dataclass
class PartitionedRelation:
    """lsj.py:71-80: worker w owns ranges[w] (device arrays)."""

    keys: torch.Tensor
    payloads: torch.Tensor
    ranges: list
    histogram: np.ndarray
    prefix_sums: np.ndarray
    overflow_total: int = 0


@dataclass
class SortedRelation:
    """lsj.py:83-92 plus the device layout: interleaved (key, payload)
    ``pairs`` in key order, bucket bounds ``starts`` of ``lmodel``'s bins."""

    pairs: torch.Tensor
    starts: torch.Tensor
    lmodel: LsjModel
    scale: int
    model_tag: tuple
    worker_ranges: list = field(default_factory=list)
    stats: SortStats = field(default_factory=SortStats)
    diag: dict = field(default_factory=dict)

    @property
    def model(self) -> RecursiveModelIndex:
        return self.lmodel.rmi

    @property
    def keys(self) -> torch.Tensor:
        return self.pairs[0::2]

    @property
    def payloads(self) -> torch.Tensor:
        return self.pairs[1::2]

    @property
    def bucket_bounds(self) -> torch.Tensor:
        """Bounds of the reference's buckets partition_index(model, key,
        scale) in the sorted output (lsj.py:302-305)."""
        return _ref_bounds(self.pairs, self.model, self.scale)


def _ref_bounds(pairs: torch.Tensor, rmi: RecursiveModelIndex, P: int) -> torch.Tensor:
    n = pairs.numel() // 2
    out = torch.empty(P + 1, dtype=torch.int64, device=pairs.device)
    c = rmi.c_struct()
    _lib.check(_lib.lib().lj_lsj_ref_bounds(ctypes.byref(c), _lib.ptr(pairs), n, P, _lib.ptr(out),
                                            _lib.stream_ptr()), "lsj_ref_bounds")
    return out


def _sort_stats(bounds: torch.Tensor) -> SortStats:
    """Comparator / partition counters of the reference's padded bitonic
    networks over the buckets with these bounds (lsj.py:250-286)."""
    sizes = (bounds[1:] - bounds[:-1]).to(torch.int64)
    nz = sizes[sizes > 0]
    if nz.numel() == 0:
        return SortStats()
    e = torch.ceil(torch.log2(nz.to(torch.float64))).to(torch.int64)
    width = torch.ones_like(e) << e
    comps = int((width * e * (e + 1) // 4).sum().item())
    return SortStats(comparator_count=comps, partitions_sorted=int(nz.numel()))


SAMPLERS = ("device", "reference")


def _sample_sorted(relation: Relation, sample_rate: float, seed: int, sampler: str = "device") -> torch.Tensor:
    """The sorted model-fit sample.  "device": one key per stratum at a
    counter-drawn offset (lj_lsj_sample).  "reference": the reference's own
    positions, numpy default_rng(seed).choice(n, total, replace=False)
    (lsj.py:119-120) drawn on the host and gathered on the device -- the
    reference's model, hence its bucket counters (comparator_count,
    partitions_sorted); the join result is the same with either."""
    if sampler not in SAMPLERS:
        raise ValueError(f"sampler must be one of {SAMPLERS}")
    n = len(relation)
    total = int(round(sample_rate * n))
    if total == 0:
        o = unsigned_order(relation.keys)
        lo, hi = torch.aminmax(o)
        return torch.stack([lo, hi]) ^ (-(2**63))
    if sampler == "reference":
        pos = np.random.default_rng(seed).choice(n, size=total, replace=False)
        picked = relation.keys[torch.from_numpy(pos.astype(np.int64)).to(relation.device)]
        return unsigned_order(torch.sort(unsigned_order(picked)).values)
    lib = _lib.lib()
    sample = torch.empty(total, dtype=torch.int64, device=relation.device)
    ws = _lib.workspace(lib.lj_lsj_sample_workspace_bytes(total), relation.device)
    # (interleaved records: the keys are every second word)
    base, stride = (relation.records, 2) if isinstance(relation, RecordRelation) else (relation.keys, 1)
    _lib.check(lib.lj_lsj_sample_strided(_lib.ptr(base), stride, n, total, int(seed) & (2**64 - 1), _lib.ptr(sample),
                                         _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "lsj_sample")
    return sample


def sample_train(relation: Relation, sample_rate: float, workers: int, seed: int,
                 fanout: int | None = None) -> RecursiveModelIndex:
    """lsj.py:95-130: the relation's CDF model fitted on a ~sample_rate
    sample (independent of ``workers``).  The sample is stratified (one key
    per stratum at a counter-drawn offset) instead of numpy's
    Generator.choice; any sample gives the same join (models are monotone)."""
    return prepare_model(relation, sample_rate, seed, fanout)[0]


def prepare_model(relation: Relation, sample_rate: float, seed: int, fanout: int | None = None,
                  nbins: int | None = None, sampler: str = "device") -> tuple[RecursiveModelIndex, LsjModel]:
    n = len(relation)
    if n == 0:
        raise ValueError("cannot sample an empty relation")
    if not 0.0 < sample_rate <= 1.0:
        raise ValueError("sample_rate must be in (0, 1]")
    sample = _sample_sorted(relation, sample_rate, seed, sampler)
    total = int(round(sample_rate * n))
    if total == 0:
        rmi = RecursiveModelIndex(fanout=1).fit(sample)
    else:
        if fanout is None:
            fanout = min(1000, max(1, total // 8))
        rmi = RecursiveModelIndex(fanout=fanout).fit(sample)
    return rmi, LsjModel.from_sample(rmi, sample, nbins or default_bins(n))


def _as_lsj_model(model, n: int) -> LsjModel:
    if isinstance(model, LsjModel):
        return model
    return LsjModel.uniform(model, default_bins(n))


def _partition(keys, payloads, lm: LsjModel):
    lib = _lib.lib()
    n = keys.numel()
    pairs = torch.empty(2 * max(n, 1), dtype=torch.int64, device=keys.device)
    starts = torch.empty(lm.nbins + 1, dtype=torch.int64, device=keys.device)
    ws = _lib.workspace(lib.lj_lsj_partition_workspace_bytes(n, lm.nbins), keys.device)
    c = lm.c_struct()
    _lib.check(lib.lj_lsj_partition(ctypes.byref(c), _lib.ptr(keys), _lib.ptr(payloads), n, _lib.ptr(pairs),
                                    _lib.ptr(starts), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "lsj_partition")
    return pairs, starts


def _regions_ok(keys, payloads, lm: LsjModel) -> bool:
    """The one-pass partition needs the bulk-copy ring (16-B aligned columns)
    and the key-range bins in shared memory (<= 2048 bins)."""
    return (lm.nbins <= 2048 and keys.numel() < 0xFFFFFFFF and keys.data_ptr() % 16 == 0
            and payloads.data_ptr() % 16 == 0 and not os.environ.get("LJ_LSJ_EXACT_PARTITION"))


def _partition_regions(keys, payloads, lm: LsjModel):
    """lj_lsj_partition_regions: ONE pass into estimated-capacity regions
    (no exact counting pass) -> (pairs with gaps, reg[2 nbins + 2])."""
    lib = _lib.lib()
    n = keys.numel()
    cap = lib.lj_lsj_partition_regions_capacity(n, lm.nbins)
    pairs = torch.empty(2 * max(cap, 1), dtype=torch.int64, device=keys.device)
    reg = torch.empty(2 * lm.nbins + 2, dtype=torch.int64, device=keys.device)
    ws = _lib.workspace(lib.lj_lsj_partition_regions_workspace_bytes(n, lm.nbins), keys.device)
    c = lm.c_struct()
    _lib.check(lib.lj_lsj_partition_regions(ctypes.byref(c), _lib.ptr(keys), _lib.ptr(payloads), n, _lib.ptr(pairs),
                                            _lib.ptr(reg), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
               "lsj_partition_regions")
    return pairs, reg


def _records_ok(rel: RecordRelation, lm: LsjModel) -> bool:
    return (lm.nbins <= 2048 and len(rel) < 0xFFFFFFFF and rel.records.data_ptr() % 16 == 0
            and not os.environ.get("LJ_LSJ_EXACT_PARTITION"))


def _partition_regions_rec(records, lm: LsjModel):
    """lj_lsj_partition_regions_rec: the one-pass regions straight from
    interleaved records (no conversion to columns)."""
    lib = _lib.lib()
    n = records.shape[0]
    cap = lib.lj_lsj_partition_regions_capacity(n, lm.nbins)
    pairs = torch.empty(2 * max(cap, 1), dtype=torch.int64, device=records.device)
    reg = torch.empty(2 * lm.nbins + 2, dtype=torch.int64, device=records.device)
    ws = _lib.workspace(lib.lj_lsj_partition_regions_workspace_bytes(n, lm.nbins), records.device)
    c = lm.c_struct()
    _lib.check(lib.lj_lsj_partition_regions_rec(ctypes.byref(c), _lib.ptr(records), n, _lib.ptr(pairs), _lib.ptr(reg),
                                                _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
               "lsj_partition_regions_rec")
    return pairs, reg


def _sort_regions(pairs_in, reg, lm: LsjModel, n: int):
    """K8 over one-pass regions -> (sorted pairs [2n], dense bin starts
    [nbins + 1], device sort counters)."""
    lib = _lib.lib()
    out = torch.empty(2 * max(n, 1), dtype=torch.int64, device=pairs_in.device)
    starts = torch.empty(lm.nbins + 1, dtype=torch.int64, device=pairs_in.device)
    ws = _lib.workspace(lib.lj_lsj_sort_workspace_bytes(n, lm.nbins), pairs_in.device)
    st = torch.zeros(4, dtype=torch.int64, device=pairs_in.device)
    c = lm.c_struct()
    _lib.check(lib.lj_lsj_sort_regions(ctypes.byref(c), _lib.ptr(pairs_in), _lib.ptr(out), n, _lib.ptr(reg),
                                       _lib.ptr(starts), _lib.ptr(ws), ws.numel(), _lib.ptr(st), _lib.stream_ptr()),
               "lsj_sort_regions")
    return out, starts, st


def _partition_sort(keys, payloads, lm: LsjModel, n: int):
    """Partition + per-bucket sort of one relation -> (sorted pairs, dense
    bin starts, sort counters): the one-pass regions when the columns allow
    them, else the exact partition."""
    if _regions_ok(keys, payloads, lm):
        pairs, reg = _partition_regions(keys, payloads, lm)
        return _sort_regions(pairs, reg, lm, n)
    pairs, starts = _partition(keys, payloads, lm)
    out, st = _sort(pairs, starts, lm, n)
    return out, starts, st


SORT_DIAG = ("oversized_sub_buckets", "bitonic_fallbacks", "big_sorted_sub_buckets", "global_sorted_sub_buckets")


def _sort(pairs_in, starts, lm: LsjModel, n: int):
    """K8 (asynchronous): -> (sorted pairs, device int64[4] sort counters;
    see SORT_DIAG and ``sort_diag``)."""
    lib = _lib.lib()
    out = torch.empty_like(pairs_in)
    ws = _lib.workspace(lib.lj_lsj_sort_workspace_bytes(n, lm.nbins), pairs_in.device)
    st = torch.zeros(4, dtype=torch.int64, device=pairs_in.device)
    c = lm.c_struct()
    _lib.check(lib.lj_lsj_sort(ctypes.byref(c), _lib.ptr(pairs_in), _lib.ptr(out), n, _lib.ptr(starts),
                               _lib.ptr(ws), ws.numel(), _lib.ptr(st), _lib.stream_ptr()), "lsj_sort")
    return out, st


def sort_diag(st) -> dict:
    """The sort counters as a dict (reads the device words)."""
    if isinstance(st, dict):
        return st
    v = st.cpu().tolist() if isinstance(st, torch.Tensor) else [0, 0, 0, 0]
    return dict(zip(SORT_DIAG, (int(x) for x in v)))


def sort_relation(keys, payloads, model, scale: int, workers: int = 1) -> SortedRelation:
    """Partition by the model and sort every bucket (lsj.py:242-313).
    ``model`` is a RecursiveModelIndex (reference-style uniform buckets) or
    an LsjModel (equi-depth bins)."""
    k = to_device_u64(keys)
    p = to_device_u64(payloads)
    n = k.numel()
    lm = _as_lsj_model(model, n)
    pairs, starts = _partition(k, p, lm)
    diag = {}
    if n:
        pairs, diag = _sort(pairs, starts, lm, n)
    srt = SortedRelation(pairs[: 2 * n], starts, lm, scale, (lm.tag, scale), diag=diag)
    bb = _ref_bounds(srt.pairs, lm.rmi, scale) if n else torch.zeros(scale + 1, dtype=torch.int64, device=k.device)
    srt.stats = _sort_stats(bb)
    if workers > 1:
        cw = scale // workers
        wb = bb[::cw].cpu().tolist()
        srt.worker_ranges = [(int(wb[w]), int(wb[w + 1])) for w in range(workers)]
    else:
        srt.worker_ranges = [(0, n)]
    return srt


def range_partition(relation: Relation, model: RecursiveModelIndex, workers: int,
                    config: LsjConfig) -> PartitionedRelation:
    """lsj.py:133-209: worker of a key = partition_index(model, key, p_eff)
    // (p_eff / workers) == partition_index(model, key, workers) (nested
    floor division); one device partition into the worker ranges.  The
    histogram is the reference's workers x workers matrix (input chunk w,
    chunk_bounds semantics, by target t), prefix_sums its write offsets;
    the order inside a range is unspecified (the multiset is the
    reference's, and so are the ranges)."""
    from .models import partition_index
    from .util import chunk_bounds

    n = len(relation)
    lm = LsjModel.uniform(model, workers)
    pairs, starts = _partition(relation.keys, relation.payloads, lm)
    st = starts.cpu().tolist()
    ranges = [(int(st[w]), int(st[w + 1])) for w in range(workers)]
    hist = np.zeros((workers, workers), dtype=np.int64)
    if n:
        target = partition_index(model, relation.keys, workers)
        b = chunk_bounds(n, workers)
        chunk = torch.repeat_interleave(torch.arange(workers, device=target.device),
                                        torch.as_tensor(np.diff(b), device=target.device))
        hist = torch.bincount(chunk * workers + target, minlength=workers * workers).reshape(workers, workers)
        hist = hist.cpu().numpy().astype(np.int64)
    totals = hist.sum(axis=0)
    target_starts = np.concatenate(([0], np.cumsum(totals)))[:-1]
    offsets = target_starts + np.cumsum(hist, axis=0) - hist
    return PartitionedRelation(pairs[0 : 2 * n : 2].contiguous(), pairs[1 : 2 * n : 2].contiguous(), ranges, hist,
                               offsets)


def cdf_bitonic_sort(keys, payloads, model, num_partitions: int):
    """lsj.py:242-286 -> (sorted keys, payloads, SortStats) as device arrays."""
    k = to_device_u64(keys)
    p = to_device_u64(payloads)
    if k.numel() == 0:
        return k.clone(), p.clone(), SortStats()
    srt = sort_relation(k, p, model, num_partitions)
    return srt.keys.contiguous(), srt.payloads.contiguous(), srt.stats


def _sort_phase(part: PartitionedRelation, model, scale: int, workers: int) -> SortedRelation:
    srt = sort_relation(part.keys, part.payloads, model, scale, workers)
    srt.worker_ranges = part.ranges
    return srt


def chunked_join(r_sorted: SortedRelation, s_sorted: SortedRelation, model_r, scale_r: int, workers: int = 1,
                 materialize: bool = False) -> JoinResult:
    """lsj.py:316-370: each sorted S tile against the R window found through
    R's model; guarded like the reference (lsj.py:329-332)."""
    if r_sorted.model_tag != (model_r.tag, scale_r):
        raise ModelMismatchError("R was bucketed under a different model or scale than the join received")
    return _join(r_sorted, s_sorted, materialize)


def _join(r_sorted: SortedRelation, s_sorted: SortedRelation, materialize: bool) -> JoinResult:
    lib = _lib.lib()
    nr = r_sorted.pairs.numel() // 2
    ns = s_sorted.pairs.numel() // 2
    dev = s_sorted.pairs.device
    c = r_sorted.lmodel.c_struct()
    args = (ctypes.byref(c), _lib.ptr(r_sorted.pairs), nr, _lib.ptr(r_sorted.starts), _lib.ptr(s_sorted.pairs), ns)
    ws = _lib.workspace(lib.lj_lsj_join_workspace_bytes(ns), dev)
    tail = (_lib.ptr(ws), ws.numel(), _lib.stream_ptr())
    if not materialize:
        out = torch.zeros(4, dtype=torch.int64, device=dev)
        _lib.check(lib.lj_lsj_join(*args, 0, None, None, None, None, _lib.ptr(out), 0, *tail), "lsj_join")
        return JoinResult(words=out)
    counts = torch.empty(max(ns, 1), dtype=torch.int64, device=dev)
    _lib.check(lib.lj_lsj_join(*args, 1, _lib.ptr(counts), None, None, None, None, 0, *tail), "lsj_join")
    offsets, total = exclusive_offsets(counts[:ns])
    pr = torch.empty(total, dtype=torch.int64, device=dev)
    ps = torch.empty(total, dtype=torch.int64, device=dev)
    if total:
        _lib.check(lib.lj_lsj_join(*args, 2, None, _lib.ptr(offsets), _lib.ptr(pr), _lib.ptr(ps), None, 0, *tail),
                   "lsj_join")
    return JoinResult(pr, ps)


def lsj_join(r: Relation | RecordRelation, s: Relation | RecordRelation, config: LsjConfig | None = None,
             materialize: bool = False, models: tuple | None = None, counters: bool = True, sampler: str = "device"):
    """lsj.py:373-405: the full learned sort-join -> (JoinResult,
    PhaseBreakdown).  Phase times are CUDA-event times on the stream.
    A ``RecordRelation`` (interleaved records, e.g. a shuffle's receive
    buffer) is sampled and partitioned in place.
    ``models`` = (model_r, model_s) RMIs fitted elsewhere (e.g. the
    reference's): they are then bucketed at the reference's uniform scale."""
    config = config or LsjConfig()
    br = PhaseBreakdown()
    if len(r) == 0 or len(s) == 0:
        return JoinResult(), br
    w = config.workers
    scale = config.effective_fanout()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    if models is None:
        _, lr = prepare_model(r, config.sample_rate, config.seed, config.model_fanout, sampler=sampler)
        _, ls = prepare_model(s, config.sample_rate, config.seed ^ 0x5DEECE66D, config.model_fanout,
                              sampler=sampler)
    else:
        lr = _as_lsj_model(models[0], len(r))
        ls = _as_lsj_model(models[1], len(s))
    ev[1].record()
    # partition: one pass into estimated-capacity regions (no exact counting
    # pass) when the columns allow it, else the exact K6/K7
    def part(rel, lm):
        if isinstance(rel, RecordRelation):
            if _records_ok(rel, lm):
                return True, _partition_regions_rec(rel.records, lm)
            rel = rel.columns()
        fast = _regions_ok(rel.keys, rel.payloads, lm)
        return fast, (_partition_regions if fast else _partition)(rel.keys, rel.payloads, lm)

    fast_r, (pr, str_) = part(r, lr)
    fast_s, (ps, sts) = part(s, ls)
    ev[2].record()
    if fast_r:
        pr, str_, dr = _sort_regions(pr, str_, lr, len(r))
    else:
        pr, dr = _sort(pr, str_, lr, len(r))
    if fast_s:
        ps, sts, ds = _sort_regions(ps, sts, ls, len(s))
    else:
        ps, ds = _sort(ps, sts, ls, len(s))
    r_sorted = SortedRelation(pr[: 2 * len(r)], str_, lr, scale, (lr.tag, scale), diag=dr)
    s_sorted = SortedRelation(ps[: 2 * len(s)], sts, ls, scale, (ls.tag, scale), diag=ds)
    ev[3].record()
    result = chunked_join(r_sorted, s_sorted, lr.rmi, scale, w, materialize)
    ev[4].record()
    ev[4].synchronize()
    br.smpl = ev[0].elapsed_time(ev[1]) / 1e3
    br.part = ev[1].elapsed_time(ev[2]) / 1e3
    br.sort = ev[2].elapsed_time(ev[3]) / 1e3
    br.join = ev[3].elapsed_time(ev[4]) / 1e3
    if counters:
        br.sort_stats = SortStats().merge(_sort_stats(r_sorted.bucket_bounds)).merge(
            _sort_stats(s_sorted.bucket_bounds))
    if counters:
        br.extra = {"bins_r": lr.nbins, "bins_s": ls.nbins, **{f"r_{k}": v for k, v in sort_diag(dr).items()},
                    **{f"s_{k}": v for k, v in sort_diag(ds).items()}}
    return result, br


def lsj_run(r: Relation | RecordRelation, s: Relation | RecordRelation,
            config: LsjConfig | None = None) -> JoinResult:
    """lsj_join in ONE asynchronous C call (lj_lsj_run): sample, fit, bins,
    partition, sort and merge-join of both relations from one workspace,
    the root of each model kept on the device.  -> JoinResult of the
    device words (the same checksum as ``lsj_join``)."""
    config = config or LsjConfig()
    dev = s.keys.device if len(s) else r.keys.device
    out = torch.zeros(4, dtype=torch.int64, device=dev)
    if len(r) == 0 or len(s) == 0:
        return JoinResult(words=out)
    lib = _lib.lib()
    ws = _lib.workspace(lib.lj_lsj_run_workspace_bytes(len(r), len(s), float(config.sample_rate)), dev)
    if isinstance(r, RecordRelation) or isinstance(s, RecordRelation):
        # lj_lsj_run_rec: both sides as interleaved records, read in place
        rr = r.records if isinstance(r, RecordRelation) else torch.stack([r.keys, r.payloads], dim=1)
        sr = s.records if isinstance(s, RecordRelation) else torch.stack([s.keys, s.payloads], dim=1)
        _lib.check(lib.lj_lsj_run_rec(_lib.ptr(rr), len(r), _lib.ptr(sr), len(s), float(config.sample_rate),
                                      int(config.seed) & (2**64 - 1), _lib.ptr(out), _lib.ptr(ws), ws.numel(),
                                      _lib.stream_ptr()), "lsj_run_rec")
        return JoinResult(words=out)
    _lib.check(lib.lj_lsj_run(_lib.ptr(r.keys), _lib.ptr(r.payloads), len(r), _lib.ptr(s.keys), _lib.ptr(s.payloads),
                              len(s), float(config.sample_rate), int(config.seed) & (2**64 - 1), _lib.ptr(out),
                              _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "lsj_run")
    return JoinResult(words=out)
