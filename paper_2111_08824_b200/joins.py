"""The drop-in boundary: the reference's runner registry (bench.py:277-318)
for the learned-join hot paths, backed by the CUDA library.

Every runner has the reference signature
``fn(r, s, workers, opts) -> (JoinResult, PhaseBreakdown, runtime_s)``.
``workers`` is the share-nothing unit: S is cut into ``workers`` chunks
with ``chunk_bounds`` exactly like the reference (bench.py:111-125), each
chunk probed on the device, partial checksums accumulated on device.  (Across
GPUs the unit is one process per GPU: see ``dist.py``.)  Index builds are
untimed, as in the reference (bench.py:138-144,202-209); LSJ is timed end to
end.  Results come back as device-reduced checksums; ``opts["materialize"]``
returns the pairs themselves (reference ``JoinResult`` semantics).
"""

from __future__ import annotations

import json
import time
from dataclasses import dataclass

import torch

from .buffers import DEFAULT_BUFFER_CAP, schedule_leaf_switches
from .data import Relation
from .gapped import GappedRmiIndex
from .learned_hash import SplineHashIndex
from .results import JoinResult, PhaseBreakdown
from .util import chunk_bounds

DEFAULT_OPTS = {
    "gap_factor": 4.0,
    "rmi_fanout": 1000,
    "buffer_cap": DEFAULT_BUFFER_CAP,
    "spline_error": 32,
    "radix_bits": 18,
    "table_factor": 4.0,
    "bucket_size": 4,
    "sample_rate": 0.01,
    "hash_sample_rate": 0.02,
    "fanout": 10000,
    "swwc": True,
    "passes": 2,
    "bits_per_pass": 6,
    "seed": 42,
    # GPU-only knobs (absent from the reference)
    "materialize": False,
    "counters": True,
    "lsj_sampler": "device",  # "reference": numpy Generator.choice positions -> the reference's bucket counters
}


@dataclass
class BenchReport:
    """bench.py:46-71 one JSON object per run, plus the checksum."""

    algorithm: str
    dataset: dict
    workers: int
    config: dict
    runtime_s: float
    throughput: float
    result_count: int
    breakdown: dict
    repetition: int = 0
    checksum: tuple = (0, 0, 0)

    def to_json(self) -> str:
        return json.dumps({
            "algorithm": self.algorithm, "dataset": self.dataset, "workers": self.workers,
            "config": self.config, "runtime_s": self.runtime_s, "throughput": self.throughput,
            "result_count": self.result_count, "repetition": self.repetition, "breakdown": self.breakdown,
            "checksum_sum": self.checksum[1], "checksum_xor": self.checksum[2],
        })


def _timed(fn):
    """Wall time of a device-synchronised call (the reference times with
    perf_counter around the whole probe, bench.py:141-143)."""
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def _chunks(n, workers):
    b = chunk_bounds(n, max(1, int(workers)))
    return [(int(b[w]), int(b[w + 1])) for w in range(len(b) - 1)]


def _materialized_probe(index, s: Relation, workers: int, br: PhaseBreakdown) -> JoinResult:
    parts = []
    for lo, hi in _chunks(len(s), workers):
        if hi == lo:
            continue
        if isinstance(index, GappedRmiIndex):
            pays, src, _ = index.search_from(None, s.keys[lo:hi], br.lookup_stats)
        else:
            pays, src = index.probe_batch(s.keys[lo:hi])
        parts.append(JoinResult(pays, s.payloads[lo:hi][src]))
    return JoinResult.concatenate(parts)


# S at least this large is grouped by index window on the device before the
# probe (the Request-Buffer analogue: K4 + staged K1s for the GRMI, the
# grouping pass + chunked probe for the learned hash); the words are
# identical, the grouped path is 3x (GRMI) / 2x (hash) faster at C2 / C3
GROUPED_MIN = 1 << 22


def _fused_probe(index, s: Relation, workers: int, grouped: bool = True) -> torch.Tensor:
    """Every S chunk probed into one device word set {count, sum, xor,
    steps}.  A host-resident S streams through ``join_checksum_host`` (H2D
    of chunk i+1 overlapped with the join of chunk i)."""
    from .streaming import join_checksum_host

    dev = (index.entries if hasattr(index, "entries") else index.slots).device
    out = torch.zeros(4, dtype=torch.int64, device=dev)
    for lo, hi in _chunks(len(s), workers):
        if hi == lo:
            continue
        buffered = grouped and hi - lo >= GROUPED_MIN
        if s.is_host:
            w = join_checksum_host(index, s.keys[lo:hi], s.payloads[lo:hi], buffered=buffered)
            out += w
        elif buffered:
            index.join_checksum_buffered(s.keys[lo:hi], s.payloads[lo:hi], out=out, accumulate=True)
        else:
            index.join_checksum(s.keys[lo:hi], s.payloads[lo:hi], out=out, accumulate=True)
    return out


def _empty():
    return JoinResult(), PhaseBreakdown(), 0.0


def _run_grmi_inlj(r, s, workers, opts):
    """bench.py:138-144: GRMI fit untimed, probe timed.  Large S is grouped
    by index window first (K4 + K1s; same words as the direct K1)."""
    index = GappedRmiIndex(opts["gap_factor"], opts["rmi_fanout"]).fit(r.to_device())
    br = PhaseBreakdown()
    if index.n == 0 or len(s) == 0:
        return JoinResult(), br, 0.0
    if opts.get("materialize"):
        s = s.to_device()
        result, runtime = _timed(lambda: _materialized_probe(index, s, workers, br))
    else:
        words, runtime = _timed(lambda: _fused_probe(index, s, workers))
        w = words.cpu().tolist()
        result = JoinResult(checksum=(int(w[0]), int(w[1]) & (2**64 - 1), int(w[2]) & (2**64 - 1)))
        br.lookup_stats.search_steps = int(w[3])
        br.lookup_stats.predictions = len(s)
    br.srch = runtime  # predict + search are one fused kernel (K1)
    if opts.get("counters", True) and len(s) and index.n:
        leaf = index.leaf_of(s.to_device().keys)  # canonical full-stream counter (bench.py:130-134)
        br.lookup_stats.leaf_switches = int((leaf[1:] != leaf[:-1]).sum().item())
    return result, br, runtime


def _run_buffered_grmi_inlj(r, s, workers, opts):
    """bench.py:147-181: request buffers -> device leaf bucketing (K4) of
    each S chunk, then the fused probe (K1s) over the bucketed chunk."""
    index = GappedRmiIndex(opts["gap_factor"], opts["rmi_fanout"]).fit(r.to_device())
    br = PhaseBreakdown()
    if index.n == 0 or len(s) == 0:
        return JoinResult(), br, 0.0
    if opts.get("materialize"):
        result, runtime = _timed(lambda: _materialized_probe(index, s.to_device(), workers, br))
    elif s.is_host:
        words, runtime = _timed(lambda: _fused_probe(index, s, workers))
        result = _words_result(words, br, len(s))
    else:
        scratch = index.bucket_scratch(max(hi - lo for lo, hi in _chunks(len(s), workers)), s.keys.device)

        def run():
            out = torch.zeros(4, dtype=torch.int64, device=s.keys.device)
            for lo, hi in _chunks(len(s), workers):
                if hi > lo:
                    index.join_checksum_buffered(s.keys[lo:hi], s.payloads[lo:hi], out=out, accumulate=True,
                                                 scratch=scratch)
            return out

        words, runtime = _timed(run)
        result = _words_result(words, br, len(s))
    if opts.get("counters", True):
        br.lookup_stats.leaf_switches = schedule_leaf_switches(index.leaf_of(s.to_device().keys), opts["buffer_cap"])
    br.join = runtime
    return result, br, runtime


def _words_result(words, br, n_s):
    w = words.cpu().tolist()
    br.lookup_stats.search_steps = int(w[3])
    br.lookup_stats.predictions = n_s
    return JoinResult(checksum=(int(w[0]) & (2**64 - 1), int(w[1]) & (2**64 - 1), int(w[2]) & (2**64 - 1)))


def _run_spline_hash_inlj(r, s, workers, opts):
    """bench.py:202-221: spline-hash fit untimed, probe timed (booked as
    pred).  Large S is grouped by index window first (same words as the
    direct K5)."""
    if len(r) == 0:
        return _empty()
    index = SplineHashIndex(opts["spline_error"], opts["radix_bits"], opts["table_factor"]).fit(r.to_device())
    br = PhaseBreakdown()
    if opts.get("materialize"):
        result, runtime = _timed(lambda: _materialized_probe(index, s.to_device(), workers, br))
    else:
        words, runtime = _timed(lambda: _fused_probe(index, s, workers))
        w = words.cpu().tolist()
        result = JoinResult(checksum=(int(w[0]) & (2**64 - 1), int(w[1]) & (2**64 - 1), int(w[2]) & (2**64 - 1)))
    br.pred = runtime
    br.lookup_stats.predictions = len(s)
    return result, br, runtime


def rmi_inlj(r_keys: torch.Tensor, r_payloads: torch.Tensor, model, s: Relation, workers: int = 1):
    """baselines.py:96-157: INLJ over the SORTED R (keys, payloads) indexed by
    a plain RMI fitted on it -> device int64[4] {count, sum, xor, steps}."""
    import ctypes

    from . import _lib

    out = torch.zeros(4, dtype=torch.int64, device=s.keys.device)
    c = model.c_struct()
    lib = _lib.lib()
    for lo, hi in _chunks(len(s), workers):
        _lib.check(lib.lj_rmi_probe(ctypes.byref(c), _lib.ptr(r_keys), _lib.ptr(r_payloads), r_keys.numel(),
                                    _lib.ptr(s.keys[lo:hi]), _lib.ptr(s.payloads[lo:hi]), hi - lo, _lib.ptr(out), 1,
                                    _lib.stream_ptr()), "rmi_probe")
    return out


def _run_rmi_inlj(r, s, workers, opts):
    """bench.py:184-192: sorted R + plain RMI fit untimed, probe timed (K12)."""
    from .models import RecursiveModelIndex
    from .util import sort_pairs, unsigned_order

    if len(r) == 0:
        return _empty()
    r, s = r.to_device(), s.to_device()
    rk, rp = sort_pairs(r.keys, r.payloads)
    model = RecursiveModelIndex(opts["rmi_fanout"]).fit(rk)
    br = PhaseBreakdown()
    words, runtime = _timed(lambda: rmi_inlj(rk, rp, model, s, workers))
    w = words.cpu().tolist()
    result = JoinResult(checksum=(int(w[0]), int(w[1]) & (2**64 - 1), int(w[2]) & (2**64 - 1)))
    if opts.get("materialize"):  # pairs on device: every S key's equal run in sorted R
        # rk is sorted as UNSIGNED u64: search in the signed view of that order
        ro, so = unsigned_order(rk), unsigned_order(s.keys)
        left = torch.searchsorted(ro, so, side="left")
        counts = torch.searchsorted(ro, so, side="right") - left
        src = torch.repeat_interleave(torch.arange(len(s), device=rk.device), counts)
        first = torch.repeat_interleave(left - (torch.cumsum(counts, 0) - counts), counts)
        slots = first + torch.arange(src.numel(), device=rk.device)
        result = JoinResult(rp[slots], s.payloads[src])
    br.lookup_stats.search_steps = int(w[3])
    br.lookup_stats.predictions = len(s)
    br.srch = runtime
    return result, br, runtime


def _run_lsj(r, s, workers, opts):
    """bench.py:224-234: LSJ timed end to end."""
    from .lsj import LsjConfig, lsj_join

    config = LsjConfig(workers=workers, sample_rate=opts["sample_rate"], fanout=opts["fanout"],
                       swwc=opts["swwc"], seed=opts["seed"])
    if (r.is_host or s.is_host) and not opts.get("materialize"):
        from .streaming import lsj_join_host

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        result = lsj_join_host(r.keys, r.payloads, s.keys, s.payloads, config)  # H2D overlapped with R's side
        _ = result.checksum
        return result, PhaseBreakdown(), time.perf_counter() - t0
    r, s = r.to_device(), s.to_device()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    result, br = lsj_join(r, s, config, materialize=bool(opts.get("materialize")),
                          counters=bool(opts.get("counters", True)), sampler=opts.get("lsj_sampler", "device"))
    _ = result.checksum  # the 3-word readback is part of the join
    return result, br, time.perf_counter() - t0


ALGORITHMS = {
    "buffered-grmi-inlj": _run_buffered_grmi_inlj,
    "grmi-inlj": _run_grmi_inlj,
    "spline-hash-inlj": _run_spline_hash_inlj,
    "lsj": _run_lsj,
    "rmi-inlj": _run_rmi_inlj,
}


def run_join(algorithm: str, r: Relation, s: Relation, workers: int = 1, opts: dict | None = None,
             dataset_echo: dict | None = None, repetition: int = 0) -> BenchReport:
    """bench.py:292-318."""
    if algorithm not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {algorithm!r}")
    merged = dict(DEFAULT_OPTS)
    if opts:
        merged.update(opts)
    result, br, runtime = ALGORITHMS[algorithm](r, s, workers, merged)
    total = len(r) + len(s)
    return BenchReport(algorithm=algorithm, dataset=dataset_echo or {"n_r": len(r), "n_s": len(s)},
                       workers=workers, config=merged, runtime_s=runtime,
                       throughput=total / runtime if runtime > 0 else 0.0, result_count=result.count,
                       breakdown=br.as_dict(), repetition=repetition, checksum=result.checksum)
