"""Request buffers (reference buffers.py) and their GPU analogue.

The reference batches probe keys per RMI leaf in fixed-capacity buffers so
that consecutive lookups touch the same index segment.  On the GPU the same
locality comes from one device pass that groups S by leaf (K4,
``lj_leaf_bucket``) before the fused probe (K1) -- see
``joins._run_buffered_grmi_inlj``.  This module keeps the reference's
planning API and its flush-by-flush ``buffered_probe`` contract (same
schedule, same delivered multiset), with the schedule computed on device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .util import as_key_tensor

DEFAULT_BUFFER_CAP = 200


@dataclass(frozen=True)
class BufferPlan:
    """buffers.py:23-41: per-buffer capacity plus the analytic size
    recurrence metadata (analysis only; no runtime role)."""

    n_models: int
    fanout: int
    cap: int = DEFAULT_BUFFER_CAP
    analytic_sizes: dict = field(default_factory=dict)
    root_buffer_size: float = 0.0
    cache_line_bytes: int = 64
    cache_capacity_bytes: int = 1 << 15


def _shrink(size, fanout):
    # divide by the fanout, exactly while it divides, fractionally after
    return size // fanout if size % fanout == 0 else size / fanout


def analytic_buffer_size(n_models: float, fanout: int) -> float:
    """buffers.py:44-49: S(n) = n + 2m S(n/m), S(x <= m) = 0."""
    if n_models <= fanout:
        return 0.0
    return n_models + 2 * fanout * analytic_buffer_size(_shrink(n_models, fanout), fanout)


def plan_buffers(n_models: int, fanout: int, cap: int = DEFAULT_BUFFER_CAP) -> BufferPlan:
    """buffers.py:52-70."""
    if n_models < 1 or fanout < 1:
        raise ValueError("n_models and fanout must be >= 1")
    if cap < 1:
        raise ValueError("cap must be >= 1")
    sizes = {}
    size = n_models
    while True:
        sizes[size] = analytic_buffer_size(size, fanout)
        if size <= fanout:
            break
        size = _shrink(size, fanout)
    return BufferPlan(n_models=n_models, fanout=fanout, cap=cap, analytic_sizes=sizes,
                      root_buffer_size=n_models + sizes[n_models])


def _leaf_groups(leaf_ids: torch.Tensor):
    order = torch.sort(leaf_ids, stable=True).indices
    sl = leaf_ids[order]
    uniq, counts = torch.unique_consecutive(sl, return_counts=True)
    starts = torch.cumsum(counts, 0) - counts
    return order, sl, uniq, counts, starts


def flush_schedule(leaf_ids: torch.Tensor, cap: int):
    """buffers.py:73-100 on device: batches of stream positions in execution
    order.  Full buffers flush when their cap-th key arrives (ordered by that
    arrival); leftovers flush at end of stream in ascending leaf order.
    Returns [(leaf, positions tensor), ...]."""
    n = leaf_ids.numel()
    if n == 0:
        return []
    order, sl, uniq, counts, starts = _leaf_groups(leaf_ids)
    occ = torch.arange(n, device=leaf_ids.device) - torch.repeat_interleave(starts, counts)
    is_end = (occ + 1) % cap == 0
    ends = torch.nonzero(is_end).flatten()               # sorted positions of full-batch ends
    end_stream_pos = order[ends]
    by_arrival = torch.argsort(end_stream_pos)
    ends = ends[by_arrival]
    batches = []
    for e, lf in zip(ends.tolist(), sl[ends].tolist()):
        batches.append((lf, order[e - cap + 1 : e + 1]))
    rem = counts % cap
    for u, c, s, r in zip(uniq.tolist(), counts.tolist(), starts.tolist(), rem.tolist()):
        if r:
            batches.append((u, order[s + c - r : s + c]))
    return batches


def schedule_leaf_switches(leaf_ids: torch.Tensor, cap: int) -> int:
    """Number of leaf changes between consecutive flushes of the canonical
    schedule (bench.py:174-179), computed without a per-flush loop."""
    n = leaf_ids.numel()
    if n == 0:
        return 0
    order, sl, uniq, counts, starts = _leaf_groups(leaf_ids)
    occ = torch.arange(n, device=leaf_ids.device) - torch.repeat_interleave(starts, counts)
    ends = torch.nonzero((occ + 1) % cap == 0).flatten()
    full = sl[ends][torch.argsort(order[ends])]
    tail = uniq[(counts % cap) != 0]
    seq = torch.cat([full, tail])
    return int((seq[1:] != seq[:-1]).sum().item()) if seq.numel() > 1 else 0


def buffered_probe(index, keys, plan: BufferPlan, sink, *, collect: str = "first"):
    """buffers.py:103-150: probe ``keys`` flush by flush through per-leaf
    request buffers; ``sink`` receives (tags, payloads, found) with
    collect="first" or (tags, payloads) with collect="all" (host arrays).
    The delivered multiset equals unbuffered lookups for any cap >= 1.

    The flush schedule is computed on the device, all flushes are searched
    in ONE device call over the keys in flush order (each flush is a
    contiguous slice of it), and the per-flush results are cut out of that
    on the host for the sink -- instead of a few small device calls and
    copies per flush."""
    from .results import LookupStats
    from .util import to_numpy_u64

    if collect not in ("first", "all"):
        raise ValueError("collect must be 'first' or 'all'")
    k = as_key_tensor(keys)
    stats = LookupStats()
    if k.numel() == 0:
        return stats
    if index.n == 0:
        tags = np.arange(k.numel(), dtype=np.int64)
        if collect == "first":
            sink(tags, np.zeros(k.numel(), dtype=np.uint64), np.zeros(k.numel(), dtype=np.bool_))
        else:
            sink(np.empty(0, dtype=np.int64), np.empty(0, dtype=np.uint64))
        return stats
    batches = flush_schedule(index.leaf_of(k), plan.cap)
    leaves = [lf for lf, _ in batches]
    stats.leaf_switches = sum(1 for a, b in zip(leaves, leaves[1:]) if a != b)
    order = torch.cat([t for _, t in batches])
    sub = LookupStats()
    pays, src, found = index.search_from(None, k[order], sub)
    stats.search_steps += sub.search_steps
    stats.predictions += sub.predictions
    tags_all = order.cpu().numpy()
    pays_h = to_numpy_u64(pays)
    src_h = src.cpu().numpy()  # non-decreasing: every probe's matches in probe order
    found_h = found.cpu().numpy()
    bounds = np.cumsum([0] + [t.numel() for _, t in batches])
    cut = np.searchsorted(src_h, bounds)  # each flush's slice of the matches
    if collect == "first":
        first = np.zeros(tags_all.size, dtype=np.uint64)
        probe, at = np.unique(src_h, return_index=True)
        first[probe] = pays_h[at]
    for b in range(len(batches)):
        lo, hi = int(bounds[b]), int(bounds[b + 1])
        if collect == "first":
            sink(tags_all[lo:hi], first[lo:hi], found_h[lo:hi])
        else:
            sink(tags_all[src_h[cut[b]:cut[b + 1]]], pays_h[cut[b]:cut[b + 1]])
    return stats
