"""Probe relations that live in host memory, transfers overlapped with the
join (INLJ).

The reference joins host-resident NumPy relations (`src/bench.py:111-144`).
On the GPU the probe side has to cross PCIe first, and at 16 B per tuple
the copy (~55 GB/s) takes ~10x longer than the probe itself (C2: 78 ms of
H2D against 7 ms of bucketing + probing).  `join_checksum_host` therefore
cuts S into chunks, copies chunk i+1 on a copy stream while chunk i is
bucketed and probed on the compute stream (double-buffered device chunks),
and accumulates the (count, sum, xor, steps) words on the device: the
result equals `join_checksum(_buffered)` over the whole S (sums wrap mod
2^64, xors commute), and the step costs about max(H2D, compute) instead of
their sum.  Keys are validated on the device per chunk (the reserved
maximum key raises ValueError once the join has finished, as
`Relation(validate=True)` would).
"""

from __future__ import annotations

import torch

DEFAULT_CHUNK = 1 << 25  # tuples per transfer (512 MiB of keys + payloads)


def _pinned(t: torch.Tensor) -> torch.Tensor:
    if t.device.type != "cpu":
        raise ValueError("join_checksum_host takes host tensors")
    return t if t.is_pinned() else t.pin_memory()


def join_checksum_host(index, keys_host: torch.Tensor, payloads_host: torch.Tensor, *, buffered: bool = True,
                       chunk: int | None = None, out: torch.Tensor | None = None,
                       scratch: dict | None = None) -> torch.Tensor:
    """(count, sum, xor, steps) of S (host int64 views of uint64 keys and
    payloads) joined with ``index`` (GappedRmiIndex or SplineHashIndex),
    copies overlapped with the probe.  ``buffered`` selects the
    Request-Buffer path (bucketing + grouped probe) per chunk."""
    if keys_host.shape != payloads_host.shape or keys_host.dim() != 1:
        raise ValueError("keys and payloads must be 1-D and of equal length")
    dev = (index.entries if hasattr(index, "entries") else index.slots).device
    n = keys_host.numel()
    out = out if out is not None else torch.zeros(4, dtype=torch.int64, device=dev)
    out.zero_()
    if n == 0 or index.n == 0:
        return out
    kh, ph = _pinned(keys_host), _pinned(payloads_host)
    c = int(min(n, chunk or DEFAULT_CHUNK))
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    bufs = [(torch.empty(c, dtype=torch.int64, device=dev), torch.empty(c, dtype=torch.int64, device=dev))
            for _ in range(2)]
    copied = [torch.cuda.Event() for _ in range(2)]
    freed = [torch.cuda.Event() for _ in range(2)]
    if buffered and scratch is None:
        scratch = index.bucket_scratch(c, dev)
    bad = torch.zeros((), dtype=torch.bool, device=dev)
    nchunks = (n + c - 1) // c
    for i in range(nchunks):
        b = i & 1
        lo, hi = i * c, min(n, (i + 1) * c)
        m = hi - lo
        with torch.cuda.stream(copy):
            if i >= 2:
                copy.wait_event(freed[b])  # chunk i-2 is probed: its buffer is free
            bufs[b][0][:m].copy_(kh[lo:hi], non_blocking=True)
            bufs[b][1][:m].copy_(ph[lo:hi], non_blocking=True)
            copied[b].record(copy)
        comp.wait_event(copied[b])
        k, p = bufs[b][0][:m], bufs[b][1][:m]
        bad |= (k == -1).any()
        if buffered:
            index.join_checksum_buffered(k, p, out=out, accumulate=True, scratch=scratch)
        else:
            index.join_checksum(k, p, out=out, accumulate=True)
        freed[b].record(comp)
    if bool(bad):
        raise ValueError("keys may not contain the reserved maximum key")
    return out


def lsj_join_host(r_keys_host: torch.Tensor, r_payloads_host: torch.Tensor, s_keys_host: torch.Tensor,
                  s_payloads_host: torch.Tensor, config=None, device=None):
    """`lsj_join` of host-resident R and S (lsj.py:373-405) with the copies
    overlapped: R and then S are copied on a copy stream; R's side (sample,
    fit, partition, sort) runs as soon as R has landed, while S is still
    crossing PCIe; then S's side and the merge-join.  Same result as
    `lsj_join` on the device-resident relations -> JoinResult."""
    from . import lsj as L
    from .data import Relation

    config = config or L.LsjConfig()
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    hs = [_pinned(t) for t in (r_keys_host, r_payloads_host, s_keys_host, s_payloads_host)]
    ds = [torch.empty(t.shape, dtype=torch.int64, device=dev) for t in hs]
    ev_r, ev_s = torch.cuda.Event(), torch.cuda.Event()
    with torch.cuda.stream(copy):
        for d, h in zip(ds[:2], hs[:2]):
            d.copy_(h, non_blocking=True)
        ev_r.record(copy)
        for d, h in zip(ds[2:], hs[2:]):
            d.copy_(h, non_blocking=True)
        ev_s.record(copy)
    comp.wait_event(ev_r)
    r = Relation(ds[0], ds[1], validate=True)
    if len(r) == 0:
        comp.wait_event(ev_s)
        return L.JoinResult()
    scale = config.effective_fanout()
    _, lr = L.prepare_model(r, config.sample_rate, config.seed, config.model_fanout)
    pr, str_, dr = L._partition_sort(r.keys, r.payloads, lr, len(r))
    comp.wait_event(ev_s)
    s = Relation(ds[2], ds[3], validate=True)
    if len(s) == 0:
        return L.JoinResult()
    _, ls = L.prepare_model(s, config.sample_rate, config.seed ^ 0x5DEECE66D, config.model_fanout)
    ps, sts, ds_ = L._partition_sort(s.keys, s.payloads, ls, len(s))
    r_sorted = L.SortedRelation(pr[: 2 * len(r)], str_, lr, scale, (lr.tag, scale), diag=dr)
    s_sorted = L.SortedRelation(ps[: 2 * len(s)], sts, ls, scale, (ls.tag, scale), diag=ds_)
    return L.chunked_join(r_sorted, s_sorted, lr.rmi, scale, config.workers)
