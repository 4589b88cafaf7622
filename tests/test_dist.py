"""Multi-process (world size 2, gloo, CPU) tests of the distributed join
protocol in paper_2111_08824_b200/dist.py: sample gathering, count
exchange, all-to-all-v, checksum reduction.  The per-rank device work is
replaced by the CPU oracle (test infrastructure), the protocol is the
product's."""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(seed=7):
    rng = np.random.default_rng(seed)
    rk = np.unique(rng.integers(0, 2**40, 30000, dtype=np.uint64))
    rk = rng.permutation(rk)
    sk = np.concatenate([rng.choice(rk, 50000), rng.integers(0, 2**40, 5000, dtype=np.uint64)])
    sk = np.concatenate([sk, np.full(3000, rk[5], np.uint64)])  # a hot duplicate key
    sk = rng.permutation(sk)
    rp = oracle.make_payloads(rk.size, 11)
    sp = oracle.make_payloads(sk.size, 12)
    return rk, rp, sk, sp


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64).copy())


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2111_08824_b200 import dist as D

    rk, rp, sk, sp = _inputs()
    rlo, rhi = D.shard_bounds(rk.size, world, rank)
    slo, shi = D.shard_bounds(sk.size, world, rank)
    r_keys, r_pay = _t(rk[rlo:rhi]), _t(rp[rlo:rhi])
    s_keys, s_pay = _t(sk[slo:shi]), _t(sp[slo:shi])

    # INLJ: replicated R, sharded S, 3-word reduction
    def probe(k, p):
        c = oracle.nlj_checksum(rk, rp, k.numpy().view(np.uint64), p.numpy().view(np.uint64))
        return torch.tensor([c[0], np.int64(np.uint64(c[1])), np.int64(np.uint64(c[2])), 0], dtype=torch.int64)

    inlj = D.inlj_join(probe, s_keys, s_pay)

    # LSJ: shared range model from the gathered samples, all-to-all-v, local join
    def model_fn(keys):
        samp = keys[:: 50].contiguous()
        allsamp = D.gather_varlen(samp)
        srt = np.sort(allsamp.numpy().view(np.uint64))
        return srt[[len(srt) * d // world for d in range(1, world)]]  # range splitters

    def partition_fn(keys, pays, splitters):
        k = keys.numpy().view(np.uint64)
        dest = np.searchsorted(splitters, k, side="right")
        order = np.argsort(dest, kind="stable")
        rec = torch.stack([keys[order], pays[order]], dim=1).contiguous()
        return rec, [int(c) for c in np.bincount(dest, minlength=world)]

    def local_join_fn(rrec, srec):
        c = oracle.smj_checksum(rrec[:, 0].numpy().view(np.uint64), rrec[:, 1].numpy().view(np.uint64),
                                srec[:, 0].numpy().view(np.uint64), srec[:, 1].numpy().view(np.uint64))
        return torch.tensor([c[0], np.int64(np.uint64(c[1])), np.int64(np.uint64(c[2])), 0], dtype=torch.int64)

    lsj, phases = D.lsj_join(r_keys, r_pay, s_keys, s_pay, group=None, model_fn=model_fn,
                             partition_fn=partition_fn, local_join_fn=local_join_fn)
    # the received ranges are disjoint and cover everything
    n_r = torch.tensor([phases["n_r_local"], phases["n_s_local"]], dtype=torch.int64)
    dist.all_reduce(n_r)
    with open(f"{out_path}.{rank}", "w") as f:
        json.dump({"inlj": list(inlj), "lsj": list(lsj), "n": n_r.tolist()}, f)
    dist.destroy_process_group()


def test_world2_inlj_and_lsj_protocol(tmp_path):
    out = str(tmp_path / "res")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    rk, rp, sk, sp = _inputs()
    want = list(oracle.smj_checksum(rk, rp, sk, sp))
    for rank in range(2):
        with open(f"{out}.{rank}") as f:
            r = json.load(f)
        assert r["inlj"] == want
        assert r["lsj"] == want
        assert r["n"] == [rk.size, sk.size]


def _wrap_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2111_08824_b200 import dist as D

    big = np.int64(np.uint64(2**64 - 3))
    words = torch.tensor([5 + rank, big, 0x0F << (8 * rank), 0], dtype=torch.int64)
    res = D.reduce_checksum(words)
    with open(f"{out_path}.{rank}", "w") as f:
        json.dump(list(res), f)
    dist.destroy_process_group()


def test_checksum_reduction_wraps_and_xors(tmp_path):
    out = str(tmp_path / "w")
    mp.spawn(_wrap_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for rank in range(2):
        with open(f"{out}.{rank}") as f:
            c, s, x = json.load(f)
        assert c == 11
        assert s == (2 * (2**64 - 3)) % 2**64
        assert x == 0x0F ^ (0x0F << 8)


@pytest.mark.parametrize("n,world", [(0, 1), (7, 3), (10**6 + 3, 8), (2_000_000_000, 8)])
def test_shard_bounds_cover(n, world):
    from paper_2111_08824_b200.dist import shard_bounds

    prev = 0
    for r in range(world):
        lo, hi = shard_bounds(n, world, r)
        assert lo == prev and hi >= lo
        prev = hi
    assert prev == n


def test_shuffle_plan_tiles_every_destination():
    """The fused shuffle's layout: for every destination, the slices the
    sources write (R then S, in source order) are disjoint and cover its
    receive buffer exactly; the capacity is the largest receive."""
    import numpy as np

    from paper_2111_08824_b200.dist import shuffle_plan

    rng = np.random.default_rng(3)
    for world in (1, 2, 3, 8):
        counts = rng.integers(0, 1000, size=(world, 2, world))
        counts[0, 1, :] = 0  # a source with nothing of S
        plans = [shuffle_plan(counts, r) for r in range(world)]
        recv_r, recv_s, cap = plans[0][0], plans[0][1], plans[0][2]
        assert cap == int((recv_r + recv_s).max())
        for d in range(world):
            cover = np.zeros(int(recv_r[d] + recv_s[d]), dtype=np.int64)
            for src in range(world):
                _, _, c2, off_r, off_s = plans[src]
                assert c2 == cap
                cover[off_r[d]:off_r[d] + counts[src, 0, d]] += 1
                cover[off_s[d]:off_s[d] + counts[src, 1, d]] += 1
            assert (cover == 1).all()


def _empty_rank_worker(rank, world, port, out_path):
    """Everything is routed to rank 0: rank 1 receives no R and no S tuples
    and must still take part in every collective (an empty local
    join used to return CPU words while the other ranks reduced over NCCL)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2111_08824_b200 import dist as D

    rk, rp, sk, sp = _inputs(9)
    rlo, rhi = D.shard_bounds(rk.size, world, rank)
    slo, shi = D.shard_bounds(sk.size, world, rank)
    r_keys, r_pay = _t(rk[rlo:rhi]), _t(rp[rlo:rhi])
    s_keys, s_pay = _t(sk[slo:shi]), _t(sp[slo:shi])

    def partition_fn(keys, pays, model):
        rec = torch.stack([keys, pays], dim=1).contiguous()
        return rec, [int(keys.numel())] + [0] * (world - 1)

    def local_join_fn(rrec, srec):
        if rrec.shape[0] == 0 or srec.shape[0] == 0:
            return torch.zeros(4, dtype=torch.int64, device=rrec.device)
        c = oracle.smj_checksum(rrec[:, 0].numpy().view(np.uint64), rrec[:, 1].numpy().view(np.uint64),
                                srec[:, 0].numpy().view(np.uint64), srec[:, 1].numpy().view(np.uint64))
        return torch.tensor([c[0], np.int64(np.uint64(c[1])), np.int64(np.uint64(c[2])), 0], dtype=torch.int64)

    res, phases = D.lsj_join(r_keys, r_pay, s_keys, s_pay, model_fn=lambda k: None, partition_fn=partition_fn,
                             local_join_fn=local_join_fn)
    with open(f"{out_path}.{rank}", "w") as f:
        json.dump({"lsj": list(res), "n": [phases["n_r_local"], phases["n_s_local"]]}, f)
    dist.destroy_process_group()


def test_world2_lsj_with_an_empty_rank(tmp_path):
    out = str(tmp_path / "e")
    mp.spawn(_empty_rank_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    rk, rp, sk, sp = _inputs(9)
    want = list(oracle.smj_checksum(rk, rp, sk, sp))
    got = []
    for rank in range(2):
        with open(f"{out}.{rank}") as f:
            got.append(json.load(f))
    assert got[0]["lsj"] == want and got[1]["lsj"] == want
    assert got[0]["n"] == [rk.size, sk.size] and got[1]["n"] == [0, 0]
