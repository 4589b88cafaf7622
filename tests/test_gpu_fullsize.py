"""GPU parity against the CPU oracle at BASELINE.json's full sizes (-m gpu).

Every configuration's device inputs equal the host generator's
(test_gpu_inputs.py), so the oracle joins the very same relations:

* C2 (2^24 join 2^28): direct K1 == K4 + staged K1s == the oracle's GRMI join
  on the same (device-fitted) model -- count, sum, xor AND search_steps.
* C3 (2*10^8 join 2*10^9, the bench headline): the grouped learned-hash
  probe == the direct one == the oracle's spline-hash join over all 2*10^9
  probes (host-generated S in 2^25-probe slices; sums add, xors xor).
* C4 (2^28 join 2^28): LSJ == the oracle's sort-merge join (the reference's
  ground truth, baselines.py:337-348) == the GRMI INLJ.
* C5 at the largest one-GPU scale (2.5*10^8 per side): the distributed LSJ
  path on a one-rank group and the local LSJ == the oracle's sort-merge join.
"""

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
MASK = (1 << 64) - 1


@pytest.fixture(scope="module")
def lj():
    import paper_2111_08824_b200 as lj

    return lj


def _words(t):
    return tuple(int(v) & MASK for v in t.cpu().tolist())


def _free():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def test_config2_full_against_oracle(lj):
    from paper_2111_08824_b200 import configs

    inp = configs.config2()
    o = dict(lj.DEFAULT_OPTS, **inp.opts)
    idx = lj.GappedRmiIndex(o["gap_factor"], o["rmi_fanout"]).fit(inp.r)
    direct = _words(idx.join_checksum(inp.s.keys, inp.s.payloads))
    buffered = _words(idx.join_checksum_buffered(inp.s.keys, inp.s.payloads))
    assert buffered == direct
    assert idx.stage_image() is not None  # the full-size path stages through the image
    rk, rp = inp.r.numpy()
    sk, sp = inp.s.numpy()
    m = idx.rmi
    om = oracle.Rmi(m.root_slope, m.root_intercept, m.trained_len, m.leaf_slope, m.leaf_intercept, m.clamp_lo,
                    m.clamp_hi, m.err_lo, m.err_hi)
    og = oracle.grmi_build(rk, rp, o["gap_factor"], o["rmi_fanout"], model=om)
    want = oracle.grmi_join(og, sk, sp)
    assert direct == tuple(v & MASK for v in want)  # count, sum, xor, search_steps
    assert want[0] == int(round(0.95 * len(inp.s)))  # every hit matches once (R unique), misses never
    del idx, inp
    _free()


def test_config3_full_against_oracle(lj):
    import oracle.gen as hg
    from paper_2111_08824_b200 import configs

    inp = configs.config3()
    o = dict(lj.DEFAULT_OPTS, **inp.opts)
    idx = lj.SplineHashIndex(o["spline_error"], o["radix_bits"], o["table_factor"]).fit(inp.r)
    grouped = _words(idx.join_checksum_buffered(inp.s.keys, inp.s.payloads))
    direct = _words(idx.join_checksum(inp.s.keys, inp.s.payloads))
    assert grouped == direct
    assert grouped[0] == len(inp.s)  # every probe is an R key, R unique
    n_s = len(inp.s)
    del idx, inp
    _free()
    host = hg.config3()
    oi = oracle.spline_hash_build(host.rk, host.rp, o["spline_error"], o["radix_bits"], o["table_factor"])
    c = s = x = 0
    step = 1 << 25
    for lo in range(0, n_s, step):
        w = oracle.spline_hash_join(oi, *host.s_slice(lo, min(n_s, lo + step)))
        c, s, x = c + w[0], (s + w[1]) & MASK, x ^ w[2]
    assert grouped[:3] == (c, s, x)


def test_config4_full_against_oracle(lj):
    from paper_2111_08824_b200 import configs

    inp = configs.config4()
    o = dict(lj.DEFAULT_OPTS, **inp.opts)
    res, _ = lj.lsj_join(inp.r, inp.s, lj.LsjConfig(fanout=o["fanout"], sample_rate=o["sample_rate"]))
    assert res.checksum[0] == len(inp.s)  # R unique, S drawn from R
    want = tuple(oracle.smj_checksum(*inp.r.numpy(), *inp.s.numpy()))
    assert res.checksum == want
    idx = lj.GappedRmiIndex(2.0, 1 << 16).fit(inp.r)
    assert _words(idx.join_checksum(inp.s.keys, inp.s.payloads))[:3] == want
    del idx, inp
    _free()


def test_config5_one_gpu_scale_against_oracle(lj, tmp_path):
    import torch.distributed as dist

    from paper_2111_08824_b200 import configs
    from paper_2111_08824_b200 import dist as ljdist

    inp = configs.config5(scale=3)  # R = S = 2.5*10^8
    want = tuple(oracle.smj_checksum(*inp.r.numpy(), *inp.s.numpy()))
    cfg = lj.LsjConfig(fanout=4096, sample_rate=0.01)
    res, _ = lj.lsj_join(inp.r, inp.s, cfg)
    assert res.checksum == want
    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        (c, s, x), _ = ljdist.lsj_join(inp.r.keys, inp.r.payloads, inp.s.keys, inp.s.payloads, cfg)
        ljdist._SYMM.clear()
    finally:
        dist.destroy_process_group()
    assert (c, s, x) == want
    del inp
    _free()
