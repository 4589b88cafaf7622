"""Multi-GPU execution of the learned joins: one process per GPU,
``torch.distributed`` (NCCL on the GPUs, gloo in the CPU tests).

INLJ: every rank holds the same R index (built untimed, as the
reference builds its index before timing) and probes its own contiguous S
shard (``shard_bounds`` = the reference's ``chunk_bounds`` unit, one GPU per
worker).  The only collective is the 3-word checksum reduction.

LSJ: one shared model, fitted on the union of the ranks' R samples,
range-partitions both relations into ``world`` contiguous key ranges
(equi-depth over the sample); per-destination counts are exchanged, then an
all-to-all-v moves the tuples (the path's one real exchange step); each rank
then runs the single-GPU LSJ on its key range, and the checksums are reduced.

The device work is injected (``partition_fn`` / ``local_join_fn``) so the
host-side protocol -- sample gathering, count exchange, split sizes,
all-to-all, checksum reduction -- is exercised by world-size-2 gloo tests on
the CPU with the oracle as the local stand-in; on GPUs the defaults call the
CUDA library.
"""

from __future__ import annotations

import ctypes
import os
import time

import numpy as np
import torch
import torch.distributed as dist

MASK = (1 << 64) - 1


def rank_world(group=None) -> tuple[int, int]:
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard of rank (util.py:62-64 chunk_bounds semantics)."""
    step = n / world
    lo = int(rank * step)
    hi = n if rank == world - 1 else int((rank + 1) * step)
    return lo, hi


def reduce_checksum(words: torch.Tensor, group=None) -> tuple[int, int, int]:
    """Combine per-rank {count, sum, xor, ...} int64 words: count and sum
    add (int64 wraps mod 2^64, as the checksum's sum does), xor is gathered
    and folded (collectives have no XOR reduction)."""
    rank, world = rank_world(group)
    w = words[:3].clone()
    if world == 1:
        v = w.cpu().tolist()
        return int(v[0]), int(v[1]) & MASK, int(v[2]) & MASK
    sums = w[:2].contiguous()
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    xs = [torch.empty_like(w[2:3]) for _ in range(world)]
    dist.all_gather(xs, w[2:3].contiguous(), group=group)
    x = 0
    for t in xs:
        x ^= int(t.item()) & MASK
    s = sums.cpu().tolist()
    return int(s[0]), int(s[1]) & MASK, x


def gather_varlen(t: torch.Tensor, group=None) -> torch.Tensor:
    """Concatenate a 1-D tensor of per-rank length across ranks (rank order)."""
    rank, world = rank_world(group)
    if world == 1:
        return t
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    sizes = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes)
    pad = torch.zeros(m, dtype=t.dtype, device=t.device)
    pad[: t.numel()] = t
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])


def exchange(records: torch.Tensor, send_counts: list[int], group=None) -> torch.Tensor:
    """All-to-all-v of records grouped by destination rank.

    ``records``: [n, 2] int64 (key, payload) ordered by destination;
    ``send_counts[d]`` records go to rank d.  Returns the records received,
    ordered by source rank."""
    rank, world = rank_world(group)
    if world == 1:
        return records
    dev = records.device
    sc = torch.tensor(send_counts, dtype=torch.int64, device=dev)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(v) for v in rc.cpu().tolist()]
    flat = records.reshape(-1).contiguous()
    out = torch.empty(2 * sum(recv_counts), dtype=flat.dtype, device=dev)
    dist.all_to_all_single(out, flat, [2 * c for c in recv_counts], [2 * c for c in send_counts], group=group)
    return out.view(-1, 2)


# ---------------------------------------------------------------- INLJ


def inlj_join(probe_fn, s_keys: torch.Tensor, s_payloads: torch.Tensor, group=None):
    """Sharded INLJ: probe_fn(keys, payloads) -> int64 words on this rank's
    S shard (replicated index), then the checksum reduction."""
    words = probe_fn(s_keys, s_payloads)
    return reduce_checksum(words, group)


# ---------------------------------------------------------------- LSJ


def _gpu_partition(keys: torch.Tensor, payloads: torch.Tensor, model, world: int):
    """Range-partition (key, payload) into `world` bins of the shared model:
    (records [n, 2] grouped by destination, counts per destination)."""
    from .lsj import _partition

    pairs, starts = _partition(keys, payloads, model)
    st = starts.cpu().tolist()
    counts = [int(st[d + 1] - st[d]) for d in range(world)]
    return pairs[: 2 * keys.numel()].view(-1, 2), counts


def _gpu_shared_model(r_keys: torch.Tensor, sample_rate: float, seed: int, world: int, group=None):
    """One model for all ranks: every rank samples its R shard, the samples
    are gathered and sorted identically everywhere, the RMI and the
    `world` equi-depth range bins are fitted on that sorted global sample
    (deterministic kernels -> the same model on every rank)."""
    from . import _lib
    from .lsj import LsjModel
    from .models import RecursiveModelIndex
    from .util import sort_pairs

    lib = _lib.lib()
    n = r_keys.numel()
    # a rank without R tuples still joins the gather, with an empty sample
    total = max(1, int(round(sample_rate * n))) if n else 0
    sample = torch.empty(total, dtype=torch.int64, device=r_keys.device)
    if total:
        ws = _lib.workspace(lib.lj_lsj_sample_workspace_bytes(total), r_keys.device)
        _lib.check(lib.lj_lsj_sample(_lib.ptr(r_keys), n, total, int(seed) & MASK, _lib.ptr(sample), _lib.ptr(ws),
                                     ws.numel(), _lib.stream_ptr()), "lsj_sample")
    allsamp = gather_varlen(sample, group)
    if allsamp.numel() == 0:
        raise ValueError("distributed LSJ: R is empty on every rank")
    srt, _ = sort_pairs(allsamp, allsamp)
    fanout = min(1000, max(1, srt.numel() // 8))
    rmi = RecursiveModelIndex(fanout).fit(srt)
    return LsjModel.from_sample(rmi, srt, world)


def shuffle_plan(counts: np.ndarray, rank: int):
    """Layout of the fused range shuffle.  counts[src, rel, dst] = tuples of
    relation rel (0 = R, 1 = S) that rank src sends to rank dst.  Every
    destination's receive buffer holds R from source 0, 1, ... then S from
    source 0, 1, ...; each source owns its slice of every destination, so
    the scatter needs no cross-GPU atomics.  Returns (recv_r[dst],
    recv_s[dst], capacity in records (the same on every rank), this rank's
    R offset in every destination, its S offset in every destination)."""
    counts = np.asarray(counts, dtype=np.int64)
    cr, cs = counts[:, 0, :], counts[:, 1, :]
    recv_r, recv_s = cr.sum(axis=0), cs.sum(axis=0)
    cap = int((recv_r + recv_s).max()) if counts.size else 0
    off_r = cr[:rank].sum(axis=0)
    off_s = recv_r + cs[:rank].sum(axis=0)
    return recv_r, recv_s, cap, off_r, off_s


_SYMM: dict = {}  # (device, group name, world) -> (symmetric receive buffer, handle)


def _pg(group):
    return group if group is not None else dist.group.WORLD


def fused_shuffle(r_keys, r_payloads, s_keys, s_payloads, model, group=None):
    """The range shuffle fused with its partition (lj_lsj_shuffle_*): exact
    per-destination counts (one all-gather of a 2 x G matrix), one symmetric-
    memory receive buffer per rank, and ONE scatter kernel per relation that
    writes every tuple straight into its destination's buffer -- NVLink P2P
    stores through the peer pointers, the all-to-all overlapped with the
    partition tile by tile.  Returns (R records [n, 2], S records [m, 2],
    buffer handle) on this rank."""
    import torch.distributed._symmetric_memory as symm

    from . import _lib

    rank, world = rank_world(group)
    lib = _lib.lib()
    dev = r_keys.device
    c = model.c_struct()
    rels = ((r_keys, r_payloads), (s_keys, s_payloads))
    cnt = torch.zeros(2, world + 1, dtype=torch.int64, device=dev)
    wss = []
    for i, (k, p) in enumerate(rels):
        n = k.numel()
        ws = _lib.workspace(lib.lj_lsj_shuffle_workspace_bytes(n, world), dev)
        _lib.check(lib.lj_lsj_shuffle_count(ctypes.byref(c), _lib.ptr(k), _lib.ptr(p), n, _lib.ptr(cnt[i]),
                                            _lib.ptr(ws), ws.numel(), _lib.stream_ptr()), "lsj_shuffle_count")
        wss.append(ws)
    allc = torch.empty(world, 2, world + 1, dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_gather_into_tensor(allc, cnt.unsqueeze(0).contiguous(), group=group)
    else:
        allc.copy_(cnt.unsqueeze(0))
    counts = allc[:, :, :world].cpu().numpy()
    recv_r, recv_s, cap, off_r, off_s = shuffle_plan(counts, rank)
    # the receive buffer is reused while it is large enough (cap is the same
    # on every rank, so every rank takes the same decision)
    # keyed by the group's NAME (a destroyed group's id() can be reused)
    key = (dev.index, getattr(_pg(group), "group_name", str(id(_pg(group)))), world)
    got = _SYMM.get(key)
    if got is None or got[0].numel() < 2 * max(cap, 1):
        buf = symm.empty(2 * max(cap, 1) + (2 * max(cap, 1)) // 8, dtype=torch.int64, device=dev)
        hdl = symm.rendezvous(buf, _pg(group))
        _SYMM[key] = (buf, hdl)
    buf, hdl = _SYMM[key]
    # peer addresses of this tensor: the symmetric blocks' bases + the
    # tensor's offset inside its block (the same on every rank)
    off0 = int(getattr(hdl, "offset", 0))
    ptrs = [int(v) + off0 for v in hdl.buffer_ptrs]
    if ptrs[rank] != buf.data_ptr():
        raise RuntimeError("symmetric memory: peer pointer of this rank does not match its buffer")
    for i, (k, p) in enumerate(rels):
        off = off_r if i == 0 else off_s
        bases = torch.tensor([ptrs[d] // 16 + int(off[d]) for d in range(world)] + [0], dtype=torch.int64, device=dev)
        _lib.check(lib.lj_lsj_shuffle_scatter(ctypes.byref(c), _lib.ptr(k), _lib.ptr(p), k.numel(), _lib.ptr(bases),
                                              _lib.ptr(wss[i]), wss[i].numel(), _lib.stream_ptr()),
                   "lsj_shuffle_scatter")
    # every rank's scatter complete before any rank reads its buffer: the
    # symmetric-memory barrier is a device-side signal / wait over the peers'
    # signal pads, ordered on the stream after the scatters (no host
    # synchronize); older handles fall back to a host sync + group barrier
    if hasattr(hdl, "barrier") and os.environ.get("LJ_SHUFFLE_HOST_BARRIER") is None:
        hdl.barrier()
    else:
        torch.cuda.current_stream(dev).synchronize()
        if world > 1:
            dist.barrier(group=group)
    rec = buf.view(-1, 2)
    nr, ns = int(recv_r[rank]), int(recv_s[rank])
    return rec[:nr], rec[nr:nr + ns], hdl


def lsj_join(r_keys, r_payloads, s_keys, s_payloads, config=None, group=None, *, model_fn=None,
             partition_fn=None, local_join_fn=None):
    """Distributed LSJ over this rank's shards of R and S.  Returns
    ((count, sum, xor), phases) -- the global checksum on every rank.

    The default shuffle is the partition followed by an NCCL all-to-all-v.
    LJ_SHUFFLE=fused selects `fused_shuffle` (partition + P2P stores into
    symmetric memory): it is checked on one GPU (a one-rank group) and by
    the layout tests, and stays opt-in until a world >= 2 parity run on a
    multi-GPU node (tests/test_gpu_multi.py) has passed."""
    from .lsj import LsjConfig

    config = config or LsjConfig()
    rank, world = rank_world(group)
    model_fn = model_fn or (lambda rk: _gpu_shared_model(rk, config.sample_rate, config.seed, world, group))
    if local_join_fn is None:
        def local_join_fn(rrec, srec):
            from . import lsj as _lsj
            from .data import RecordRelation

            # the received records are partitioned in place (no copy back to columns)
            r, s = RecordRelation(rrec), RecordRelation(srec)
            res, _ = _lsj.lsj_join(r, s, LsjConfig(workers=1, fanout=config.fanout,
                                                    sample_rate=config.sample_rate, seed=config.seed),
                                   counters=False)
            if res._words is not None:
                return res._words
            # empty local join (a rank that received no R or no S tuples):
            # the words live on the device like every other rank's, so the
            # NCCL reduction below sees a CUDA tensor on every rank
            sg = [v - (1 << 64) if v >= (1 << 63) else v for v in list(res.checksum) + [0]]
            return torch.tensor(sg, dtype=torch.int64, device=rrec.device)
    phases = {}
    fused = (partition_fn is None and r_keys.is_cuda and os.environ.get("LJ_SHUFFLE", "nccl") == "fused")
    t0 = time.perf_counter()
    model = model_fn(r_keys)
    t1 = time.perf_counter()
    hdl = None
    if fused:
        r_loc, s_loc, hdl = fused_shuffle(r_keys, r_payloads, s_keys, s_payloads, model, group)
        t2 = t3 = time.perf_counter()
    else:
        partition_fn = partition_fn or (lambda k, p, m: _gpu_partition(k, p, m, world))
        r_rec, r_cnt = partition_fn(r_keys, r_payloads, model)
        s_rec, s_cnt = partition_fn(s_keys, s_payloads, model)
        t2 = time.perf_counter()
        r_loc = exchange(r_rec, r_cnt, group)
        s_loc = exchange(s_rec, s_cnt, group)
        t3 = time.perf_counter()
    words = local_join_fn(r_loc, s_loc)
    t4 = time.perf_counter()
    del hdl  # the receive buffers stay alive until the local join is done
    res = reduce_checksum(words, group)
    phases.update(smpl=t1 - t0, part=t2 - t1, xchg=t3 - t2, local=t4 - t3, n_r_local=int(r_loc.shape[0]),
                  n_s_local=int(s_loc.shape[0]), shuffle="fused P2P" if fused else "partition + NCCL all-to-all-v")
    return res, phases


# ------------------------------------------- single-process multi-GPU (C ABI)
# The same distributed LSJ as one call over several devices of this process
# (lj_lsj_run_multi: NCCL communicators from ncclCommInitAll, one stream per
# device) -- the drop-in for the reference's `workers` when the workers are
# GPUs driven from one host thread.

_NCCL_COMMS: dict = {}


def _ptrs(vals, ctype=ctypes.c_void_p):
    return (ctype * len(vals))(*vals)


def nccl_comms(devices) -> list:
    """One NCCL communicator per device (cached per device tuple)."""
    from . import _lib

    key = tuple(int(d) for d in devices)
    if key not in _NCCL_COMMS:
        lib = _lib.lib()
        if lib.lj_nccl_available() != 1:
            raise RuntimeError("NCCL (libnccl.so.2) is not available")
        arr = (ctypes.c_void_p * len(key))()
        _lib.check(lib.lj_nccl_comm_init_all(len(key), _ptrs(key, ctypes.c_int), arr), "nccl_comm_init_all")
        _NCCL_COMMS[key] = [int(a) for a in arr]
    return _NCCL_COMMS[key]


def reduce_sums_multi(words: list) -> tuple[int, int, int]:
    """lj_reduce_sums over the devices of this process: words[d] (device
    int64[4]) all become the global (count, sum, xor)."""
    from . import _lib

    devs = [w.device.index for w in words]
    comms = nccl_comms(devs)
    lib = _lib.lib()
    ws = [torch.empty(lib.lj_reduce_sums_workspace_bytes(len(devs)), dtype=torch.uint8, device=w.device)
          for w in words]
    streams = [torch.cuda.current_stream(w.device).cuda_stream for w in words]
    _lib.check(lib.lj_reduce_sums(len(devs), _ptrs(devs, ctypes.c_int), _ptrs(comms), _ptrs(streams),
                                  _ptrs([w.data_ptr() for w in words]), _ptrs([t.data_ptr() for t in ws])),
               "reduce_sums")
    v = words[0].cpu().tolist()
    return int(v[0]), int(v[1]) & MASK, int(v[2]) & MASK


def lsj_run_multi(r_parts: list, s_parts: list, config=None, cap_factor: float = 1.5):
    """The distributed LSJ over this process's devices in one C call:
    r_parts[d] / s_parts[d] are the shards (Relations) on device d.
    -> (count, sum, xor)."""
    from . import _lib
    from .lsj import LsjConfig

    config = config or LsjConfig()
    lib = _lib.lib()
    n = len(r_parts)
    devs = [p.keys.device.index for p in r_parts]
    comms = nccl_comms(devs)
    nr = [len(p) for p in r_parts]
    ns = [len(p) for p in s_parts]
    nr_t, ns_t = sum(nr), sum(ns)
    cap_r = min(nr_t, int(cap_factor * nr_t / n) + 4096)
    cap_s = min(ns_t, int(cap_factor * ns_t / n) + 4096)
    outs = [torch.zeros(4, dtype=torch.int64, device=p.keys.device) for p in r_parts]
    streams = [torch.cuda.current_stream(p.keys.device).cuda_stream for p in r_parts]
    for _ in range(2):
        wsb = [lib.lj_lsj_run_multi_workspace_bytes(n, nr[d], ns[d], nr_t, max(cap_r, 1), max(cap_s, 1),
                                                    float(config.sample_rate)) for d in range(n)]
        ws = [torch.empty(b, dtype=torch.uint8, device=p.keys.device) for b, p in zip(wsb, r_parts)]
        recv = (ctypes.c_int64 * (2 * n))()
        rc = lib.lj_lsj_run_multi(n, _ptrs(devs, ctypes.c_int), _ptrs(comms), _ptrs(streams),
                                  _ptrs([p.keys.data_ptr() for p in r_parts]),
                                  _ptrs([p.payloads.data_ptr() for p in r_parts]), _ptrs(nr, ctypes.c_int64),
                                  _ptrs([p.keys.data_ptr() for p in s_parts]),
                                  _ptrs([p.payloads.data_ptr() for p in s_parts]), _ptrs(ns, ctypes.c_int64),
                                  max(cap_r, 1), max(cap_s, 1), float(config.sample_rate),
                                  int(config.seed) & MASK, _ptrs([o.data_ptr() for o in outs]),
                                  _ptrs([w.data_ptr() for w in ws]), _ptrs(wsb, ctypes.c_size_t), recv)
        if rc == _lib.LJ_E_WORKSPACE and any(recv):
            cap_r = max(cap_r, max(recv[2 * d] for d in range(n)))
            cap_s = max(cap_s, max(recv[2 * d + 1] for d in range(n)))
            continue
        _lib.check(rc, "lsj_run_multi")
        break
    v = outs[0].cpu().tolist()
    return int(v[0]), int(v[1]) & MASK, int(v[2]) & MASK
