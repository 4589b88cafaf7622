"""Learned sort-join on the GPU (reference lsj.py:1-405).

Per relation: a stratified sample of ``sample_rate`` (K-sample), an RMI fit
on the sorted sample (K10), a CDF partition into Pf = P*F fine buckets (K6
histogram + K7 warp-aggregated scatter), and a model-placed per-bucket sort
in shared memory (K8; oversized buckets through global memory).  The join
(K9) walks sorted S in tiles and merge-searches each tile's R window found
through R's model.  P is the reference's sort-phase scale
(``effective_fanout``); F refines it so that a fine bucket averages <= 1024
tuples (fits shared memory), and every F-th fine bound is a coarse bound,
which is what the reference's bucket_bounds / counters are computed from.

``workers`` keeps the reference's meaning for the bucket scale (P is a
multiple of it) and for ``range_partition``; on one GPU all workers' ranges
are processed by the same kernels.  Across GPUs the worker is a GPU (see
``dist.py``).  Results: the checksum (count, sum, xor) of
R.payload + S.payload over all matching pairs; pairs on request.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .data import Relation
from .models import RecursiveModelIndex, partition_index
from .results import JoinResult, PhaseBreakdown, SortStats
from .util import exclusive_offsets, to_device_u64, unsigned_order

FINE_TARGET = 1024  # mean tuples per fine bucket (shared-memory sort unit)


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
    ``pairs``, fine bucket bounds ``fine_starts`` at scale ``fine_scale``."""

    pairs: torch.Tensor
    fine_starts: torch.Tensor
    fine_scale: int
    scale: int
    model: RecursiveModelIndex
    model_tag: tuple
    worker_ranges: list = field(default_factory=list)
    stats: SortStats = field(default_factory=SortStats)

    @property
    def keys(self) -> torch.Tensor:
        return self.pairs[0::2]

    @property
    def payloads(self) -> torch.Tensor:
        return self.pairs[1::2]

    @property
    def bucket_bounds(self) -> torch.Tensor:
        """Coarse bounds at the reference's scale (every F-th fine bound)."""
        f = self.fine_scale // self.scale
        return self.fine_starts[::f].contiguous()


def _fine_scale(n: int, scale: int) -> int:
    return scale * max(1, math.ceil(n / (scale * FINE_TARGET)))


def sample_train(relation: Relation, sample_rate: float, workers: int, seed: int,
                 fanout: int | None = None) -> RecursiveModelIndex:
    """lsj.py:95-130: fit the relation's CDF model on a ~sample_rate sample
    (independent of ``workers``).  The sample is stratified (one key per
    stratum at a counter-drawn offset) instead of numpy's Generator.choice;
    any sample gives the same join result (models are monotone)."""
    n = len(relation)
    if n == 0:
        raise ValueError("cannot sample an empty relation")
    if not 0.0 < sample_rate <= 1.0:
        raise ValueError("sample_rate must be in (0, 1]")
    total = int(round(sample_rate * n))
    lib = _lib.lib()
    dev = relation.device
    if total == 0:
        o = unsigned_order(relation.keys)
        lo, hi = torch.aminmax(o)
        two = torch.stack([lo, hi]) ^ (-(2**63))
        return RecursiveModelIndex(fanout=1).fit(two)
    sample = torch.empty(total, dtype=torch.int64, device=dev)
    ws = _lib.workspace(lib.lj_lsj_sample_workspace_bytes(total), dev)
    _lib.check(lib.lj_lsj_sample(_lib.ptr(relation.keys), n, total, int(seed) & (2**64 - 1), _lib.ptr(sample),
                                 _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "lsj_sample")
    if fanout is None:
        fanout = min(1000, max(1, total // 8))
    return RecursiveModelIndex(fanout=fanout).fit(sample)


def _partition(keys, payloads, model, nbins):
    lib = _lib.lib()
    n = keys.numel()
    pairs = torch.empty(2 * max(n, 1), dtype=torch.int64, device=keys.device)
    starts = torch.empty(nbins + 1, dtype=torch.int64, device=keys.device)
    ws = _lib.workspace(lib.lj_lsj_partition_workspace_bytes(n, nbins), keys.device)
    c = model.c_struct()
    _lib.check(lib.lj_lsj_partition(ctypes.byref(c), _lib.ptr(keys), _lib.ptr(payloads), n, nbins, _lib.ptr(pairs),
                                    _lib.ptr(starts), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "lsj_partition")
    return pairs, starts


def _sort_in_place(pairs, starts, model, n, nbins):
    """K8 (+ the oversized path and the run pass) on partitioned pairs."""
    lib = _lib.lib()
    dev = pairs.device
    ws = _lib.workspace(lib.lj_lsj_sort_workspace_bytes(n, nbins), dev)
    c = model.c_struct()
    st = (ctypes.c_int64 * 2)()
    _lib.check(lib.lj_lsj_sort_buckets(ctypes.byref(c), _lib.ptr(pairs), n, nbins, _lib.ptr(starts), _lib.ptr(ws),
                                       ws.numel(), st, _lib.stream_ptr()), "lsj_sort_buckets")
    n_over = int(st[0])
    if n_over:
        seg = np.empty(n_over, dtype=np.int64)
        _lib.check(lib.lj_lsj_oversized_list_host(_lib.ptr(ws), n, n_over, seg.ctypes.data), "oversized_list")
        seg.sort()
        sb = starts.cpu().numpy()
        beg = np.ascontiguousarray(sb[seg])
        end = np.ascontiguousarray(sb[seg + 1])
        total = int((end - beg).sum())
        ows = _lib.workspace(lib.lj_lsj_sort_oversized_workspace_bytes(n_over, total), dev)
        st2 = (ctypes.c_int64 * 2)()
        _lib.check(lib.lj_lsj_sort_oversized(ctypes.byref(c), _lib.ptr(pairs), n, nbins, seg.ctypes.data,
                                             beg.ctypes.data, end.ctypes.data, n_over, _lib.ptr(ws), _lib.ptr(ows),
                                             ows.numel(), st2, _lib.stream_ptr()), "lsj_sort_oversized")
    _lib.check(lib.lj_lsj_sort_runs(_lib.ptr(pairs), n, _lib.ptr(ws), _lib.stream_ptr()), "lsj_sort_runs")
    return n_over


def _sort_stats(fine_starts: torch.Tensor, fine_scale: int, scale: int) -> SortStats:
    """Comparator / partition counters of the reference's padded bitonic
    networks at scale P (lsj.py:250-286; tests/test_lsj.py:27-32), from the
    coarse bucket sizes."""
    f = fine_scale // scale
    sizes = (fine_starts[f::f] - fine_starts[:-1:f]).to(torch.int64)
    nz = sizes[sizes > 0]
    if nz.numel() == 0:
        return SortStats()
    e = torch.ceil(torch.log2(nz.to(torch.float64))).to(torch.int64)
    width = torch.ones_like(e) << e
    comps = int((width * e * (e + 1) // 4).sum().item())
    return SortStats(comparator_count=comps, partitions_sorted=int(nz.numel()))


def sort_relation(keys, payloads, model: RecursiveModelIndex, scale: int, workers: int = 1) -> SortedRelation:
    """Partition at the fine scale and sort every bucket (lsj.py:289-313)."""
    n = keys.numel()
    fine = _fine_scale(n, scale)
    pairs, starts = _partition(keys, payloads, model, fine)
    if n:
        _sort_in_place(pairs, starts, model, n, fine)
    srt = SortedRelation(pairs[: 2 * n], starts, fine, scale, model, (model.tag, scale))
    srt.stats = _sort_stats(starts, fine, scale)
    bb = srt.bucket_bounds
    if workers > 1:
        cw = scale // workers
        wb = bb[::cw].cpu().tolist()
        srt.worker_ranges = [(int(wb[w]), int(wb[w + 1])) for w in range(workers)]
    else:
        srt.worker_ranges = [(0, n)]
    return srt


def range_partition(relation: Relation, model: RecursiveModelIndex, workers: int,
                    config: LsjConfig) -> PartitionedRelation:
    """lsj.py:133-209: each key goes to worker partition_index(model, key,
    p_eff) // (p_eff / workers) == partition_index(model, key, workers).
    Order inside a worker range is unspecified (the multiset is the
    reference's)."""
    n = len(relation)
    pairs, starts = _partition(relation.keys, relation.payloads, model, workers)
    st = starts.cpu().tolist()
    ranges = [(int(st[w]), int(st[w + 1])) for w in range(workers)]
    hist = np.diff(np.asarray(st, dtype=np.int64)).reshape(1, workers)
    return PartitionedRelation(pairs[0 : 2 * n : 2].contiguous(), pairs[1 : 2 * n : 2].contiguous(), ranges, hist,
                               np.asarray(st[:-1], dtype=np.int64).reshape(1, workers))


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
    """lsj.py:316-370: each S tile against its R window through R's model."""
    if r_sorted.model_tag != (model_r.tag, scale_r):
        raise ModelMismatchError("R was bucketed under a different model or scale than the join received")
    return _join(r_sorted, s_sorted, materialize)


def _join(r_sorted: SortedRelation, s_sorted: SortedRelation, materialize: bool) -> JoinResult:
    lib = _lib.lib()
    nr = r_sorted.pairs.numel() // 2
    ns = s_sorted.pairs.numel() // 2
    dev = s_sorted.pairs.device
    c = r_sorted.model.c_struct()
    args = (ctypes.byref(c), _lib.ptr(r_sorted.pairs), nr, r_sorted.fine_scale, _lib.ptr(r_sorted.fine_starts),
            _lib.ptr(s_sorted.pairs), ns)
    if not materialize:
        out = torch.zeros(4, dtype=torch.int64, device=dev)
        _lib.check(lib.lj_lsj_join(*args, 0, None, None, None, None, _lib.ptr(out), 0, _lib.stream_ptr()), "lsj_join")
        return JoinResult(words=out)
    counts = torch.empty(max(ns, 1), dtype=torch.int64, device=dev)
    _lib.check(lib.lj_lsj_join(*args, 1, _lib.ptr(counts), None, None, None, None, 0, _lib.stream_ptr()), "lsj_join")
    offsets, total = exclusive_offsets(counts[:ns])
    pr = torch.empty(total, dtype=torch.int64, device=dev)
    ps = torch.empty(total, dtype=torch.int64, device=dev)
    if total:
        _lib.check(lib.lj_lsj_join(*args, 2, None, _lib.ptr(offsets), _lib.ptr(pr), _lib.ptr(ps), None, 0,
                                   _lib.stream_ptr()), "lsj_join")
    return JoinResult(pr, ps)


def lsj_join(r: Relation, s: Relation, config: LsjConfig | None = None, materialize: bool = False,
             models: tuple | None = None):
    """lsj.py:373-405: the full learned sort-join -> (JoinResult,
    PhaseBreakdown).  Phase times are CUDA-event times on the stream."""
    config = config or LsjConfig()
    br = PhaseBreakdown()
    if len(r) == 0 or len(s) == 0:
        return JoinResult(), br
    w = config.workers
    scale = config.effective_fanout()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    if models is None:
        model_r = sample_train(r, config.sample_rate, w, config.seed, config.model_fanout)
        model_s = sample_train(s, config.sample_rate, w, config.seed ^ 0x5DEECE66D, config.model_fanout)
    else:
        model_r, model_s = models
    ev[1].record()
    fr, fs = _fine_scale(len(r), scale), _fine_scale(len(s), scale)
    pr, str_ = _partition(r.keys, r.payloads, model_r, fr)
    ps, sts = _partition(s.keys, s.payloads, model_s, fs)
    ev[2].record()
    over_r = _sort_in_place(pr, str_, model_r, len(r), fr)
    over_s = _sort_in_place(ps, sts, model_s, len(s), fs)
    r_sorted = SortedRelation(pr[: 2 * len(r)], str_, fr, scale, model_r, (model_r.tag, scale))
    s_sorted = SortedRelation(ps[: 2 * len(s)], sts, fs, scale, model_s, (model_s.tag, scale))
    ev[3].record()
    result = chunked_join(r_sorted, s_sorted, model_r, scale, w, materialize)
    ev[4].record()
    ev[4].synchronize()
    br.smpl = ev[0].elapsed_time(ev[1]) / 1e3
    br.part = ev[1].elapsed_time(ev[2]) / 1e3
    br.sort = ev[2].elapsed_time(ev[3]) / 1e3
    br.join = ev[3].elapsed_time(ev[4]) / 1e3
    br.sort_stats = SortStats().merge(_sort_stats(str_, fr, scale)).merge(_sort_stats(sts, fs, scale))
    br.extra = {"fine_scale_r": fr, "fine_scale_s": fs, "oversized_buckets_r": over_r, "oversized_buckets_s": over_s}
    return result, br


@dataclass(frozen=True)
class LsjCostParams:
    """lsj.py:408-430 inputs of the per-worker cost estimate (analysis only)."""

    n_r: int
    n_s: int
    s_r: int = 0
    s_s: int = 0
    p_r: int = 1
    p_s: int = 1
    o_r: int = 0
    o_s: int = 0
    workers: int = 1

    def __post_init__(self):
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.p_r < self.workers or self.p_s < self.workers:
            raise ValueError("partition counts must be >= workers")
        if not (0 <= self.o_r <= self.workers and 0 <= self.o_s <= self.workers):
            raise ValueError("overlap counts must be within [0, workers]")
