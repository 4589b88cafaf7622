"""GPU parity: the CUDA path against the reference's golden vectors and the
C oracle, through the C ABI.  Bit-exact for every integer output."""

import ctypes

import numpy as np
import pytest
import torch

import oracle
from conftest import rmi_from_fixture

pytestmark = pytest.mark.gpu

MASK = (1 << 64) - 1


@pytest.fixture(scope="module")
def lj():
    import paper_2111_08824_b200 as lj

    return lj


def _np(t):
    from paper_2111_08824_b200.util import to_numpy_u64

    return to_numpy_u64(t)


def _i64(t):
    return t.cpu().numpy().astype(np.int64)


def ref_rmi(lj, d, prefix=""):
    return lj.RecursiveModelIndex.from_params(
        d[prefix + "root"][0], d[prefix + "root"][1], int(d[prefix + "trained_len"]), d[prefix + "leaf_slope"],
        d[prefix + "leaf_intercept"], d[prefix + "clamp_lo"], d[prefix + "clamp_hi"], d[prefix + "err_lo"],
        d[prefix + "err_hi"])


MODEL_SETS = ["unif63", "lognorm1e12", "clusters", "seq_h", "lognorm_ref", "dups", "linear", "tiny", "single",
              "dbl_collide"]


@pytest.mark.parametrize("name", MODEL_SETS)
def test_rmi_eval_bitwise(golden, lj, name):
    """L0: models.py:112-135 + partition_index on device == reference."""
    d = golden("models")[name]
    m = ref_rmi(lj, d)
    pos, lo, hi = m.predict_many(d["probes"])
    assert np.array_equal(_i64(pos), d["pos"])
    assert np.array_equal(_i64(lo), d["lo"])
    assert np.array_equal(_i64(hi), d["hi"])
    assert np.array_equal(_i64(m.route_many(d["probes"])), d["route"])
    for P in (1, 7, 4096):
        assert np.array_equal(_i64(lj.partition_index(m, d["probes"], P)), d[f"part_{P}"])


@pytest.mark.parametrize("name", MODEL_SETS)
def test_spline_eval_bitwise(golden, lj, name):
    d = golden("models")[name]
    me, rb = int(d["sp_max_error"]), int(d["sp_radix_bits"])
    sp = lj.RadixSplineIndex(me, rb).fit(d["keys"])
    assert np.array_equal(sp.spline_keys, d["sp_keys"])
    pos, lo, hi = sp.predict_many(d["probes"])
    assert np.array_equal(_i64(pos), d["sp_pos"])
    assert np.array_equal(_i64(lo), d["sp_lo"])
    assert np.array_equal(_i64(hi), d["sp_hi"])
    n = d["keys"].size
    assert np.array_equal(_i64(lj.partition_index(sp, d["probes"], 4 * n)), d["sp_part_4n"])
    assert np.array_equal(_i64(lj.partition_index(sp, d["probes"], 3)), d["sp_part_3"])


@pytest.mark.parametrize("name", MODEL_SETS)
def test_rmi_fit_on_device_is_sound(golden, lj, name):
    """K10: bounds contain every true rank, predictions monotone, clamps
    equal the reference's (they are integer segment bounds)."""
    d = golden("models")[name]
    keys = d["keys"]
    m = lj.RecursiveModelIndex(int(d["fanout"])).fit(keys)
    pos, lo, hi = (_i64(t) for t in m.predict_many(keys))
    truth = np.searchsorted(keys, keys, side="left")
    assert np.all((lo <= truth) & (truth <= hi))
    assert np.all(np.diff(pos) >= 0)
    if name != "dbl_collide":
        assert np.array_equal(m.clamp_lo, d["clamp_lo"])
        assert np.array_equal(m.clamp_hi, d["clamp_hi"])
        np.testing.assert_allclose(m.leaf_slope, d["leaf_slope"], rtol=1e-6, atol=1e-12)


def test_grmi_layout_search_and_join_bitwise(golden, lj):
    """L0-L2 on every golden GRMI case, with the reference's own model:
    identical gapped arrays, slots, per-probe search results and probe
    counts, pairs, checksum and search_steps."""
    for case, d in golden("grmi").items():
        rel = lj.Relation(d["keys"], d["payloads"])
        idx = lj.GappedRmiIndex(float(d["gap"]), int(d["fanout"])).fit(rel, model=ref_rmi(lj, d))
        assert idx.slot_count == int(d["L"]), case
        assert np.array_equal(idx.gkeys, d["gkeys"]), case
        assert np.array_equal(idx.gpayloads, d["gpayloads"]), case
        assert np.array_equal(idx.bitmap, d["bitmap"]), case
        slots0 = idx.predict_slots(d["probes"])
        assert np.array_equal(_i64(slots0), d["slots0"]), case
        slot, probes = idx.search(slots0, d["probes"])
        assert np.array_equal(_i64(slot), d["out_slot"]), case
        assert np.array_equal(_i64(probes), d["out_probes"]), case
        st = lj.LookupStats()
        pays, src, found = idx.lookup_batch(d["probes"], st)
        assert np.array_equal(_np(pays), d["pairs_r"]), case
        assert np.array_equal(_i64(src), d["pairs_src"]), case
        assert np.array_equal(found.cpu().numpy(), d["found"]), case
        assert [st.search_steps, st.predictions, st.leaf_switches] == d["stats"].tolist(), case
        s = lj.Relation(d["probes"], d["probe_payloads"])
        w = idx.join_checksum(s.keys, s.payloads).cpu().tolist()
        assert (w[0], w[1] & MASK, w[2] & MASK) == tuple(int(v) for v in d["checksum"]), case
        assert w[3] == int(d["stats"][0]), case


def test_grmi_zero_payloads_use_the_bitmap(lj):
    """A real payload of 0 switches the kernel to bitmap occupancy."""
    keys = np.array([5, 5, 5, 9, 20, 21, 40], np.uint64)
    pays = np.array([0, 1, 2, 0, 4, 5, 0], np.uint64)
    idx = lj.GappedRmiIndex(2.0, 2).fit(lj.Relation(keys, pays))
    assert idx.payload_nonzero == 0
    probes = np.array([5, 9, 40, 7, 21, 5], np.uint64)
    pp = np.arange(10, 16, dtype=np.uint64)
    w = idx.join_checksum(lj.Relation(probes, pp).keys, lj.Relation(probes, pp).payloads).cpu().tolist()
    want = oracle.nlj_checksum(keys, pays, probes, pp)
    assert (w[0], w[1] & MASK, w[2] & MASK) == want
    assert sorted(idx.lookup_range(5).tolist()) == [0, 1, 2]


def test_spline_hash_build_and_probe_bitwise(golden, lj):
    for case, d in golden("spline_hash").items():
        n = d["keys"].size
        model = lj.RadixSplineIndex.from_params(d["sp_keys"], d["sp_ranks"], d["sp_radix_table"], int(d["sp_shift"]),
                                                n, int(d["max_error"]), int(d["radix_bits"]))
        rel = lj.Relation(d["keys"], d["payloads"])
        idx = lj.SplineHashIndex(int(d["max_error"]), int(d["radix_bits"]), float(d["table_factor"])).fit(rel, model)
        assert idx.table_len == int(d["table_len"]), case
        assert np.array_equal(idx._keys, d["e_keys"]), case
        assert np.array_equal(idx._payloads, d["e_payloads"]), case
        assert idx.collision_fraction() == float(d["collision_fraction"]), case
        pays, src = idx.probe_batch(d["probes"])
        assert np.array_equal(_np(pays), d["pairs_r"]), case
        assert np.array_equal(_i64(src), d["pairs_src"]), case
        s = lj.Relation(d["probes"], d["probe_payloads"])
        w = idx.join_checksum(s.keys, s.payloads).cpu().tolist()
        assert (w[0], w[1] & MASK, w[2] & MASK) == tuple(int(v) for v in d["checksum"]), case
        # own host fit picks the same spline
        own = lj.SplineHashIndex(int(d["max_error"]), int(d["radix_bits"]), float(d["table_factor"])).fit(rel)
        assert np.array_equal(own.model.spline_keys, d["sp_keys"]), case


@pytest.mark.parametrize("algo", ["grmi-inlj", "buffered-grmi-inlj", "spline-hash-inlj", "lsj", "rmi-inlj"])
@pytest.mark.parametrize("workers", [1, 4])
def test_algorithms_registry_matches_reference(golden, lj, algo, workers):
    """L2 through the drop-in boundary (bench.py:277-289): every c01-style
    case's checksum equals the reference runner's; materialised pairs equal
    the reference multiset."""
    for case, d in golden("algos").items():
        r = lj.Relation(d["r_keys"], d["r_payloads"])
        s = lj.Relation(d["s_keys"], d["s_payloads"])
        opts = dict(lj.DEFAULT_OPTS)
        res, br, rt = lj.ALGORITHMS[algo](r, s, workers, opts)
        assert res.checksum == tuple(int(v) for v in d["checksum"]), (case, algo)
        if algo != "lsj":
            assert br.lookup_stats.predictions == len(s)
        opts["materialize"] = True
        res2, _, _ = lj.ALGORITHMS[algo](r, s, workers, opts)
        assert res2.checksum == res.checksum
        want = oracle.nlj_checksum(d["r_keys"], d["r_payloads"], d["s_keys"], d["s_payloads"])
        assert res2.checksum == want


def test_config1_full_size_against_oracle(lj):
    """C1 at full size (R 2^20, S 2^22): GPU checksum and search_steps equal
    the oracle's on the same inputs and the same model."""
    from paper_2111_08824_b200 import configs

    inp = configs.config1()
    idx = lj.GappedRmiIndex(2.0, 1024).fit(inp.r)
    w = idx.join_checksum(inp.s.keys, inp.s.payloads).cpu().tolist()
    rk, rp = inp.r.numpy()
    sk, sp = inp.s.numpy()
    om = oracle.Rmi(idx.rmi.root_slope, idx.rmi.root_intercept, idx.rmi.trained_len, idx.rmi.leaf_slope,
                    idx.rmi.leaf_intercept, idx.rmi.clamp_lo, idx.rmi.clamp_hi, idx.rmi.err_lo, idx.rmi.err_hi)
    og = oracle.grmi_build(rk, rp, 2.0, 1024, model=om)
    assert np.array_equal(og.gkeys, idx.gkeys)
    want = oracle.grmi_join(og, sk, sp)
    assert (w[0], w[1] & MASK, w[2] & MASK, w[3]) == want
    assert want[0] == int(round(0.9 * (1 << 22)))  # every hit matches exactly once
    assert oracle.smj_checksum(rk, rp, sk, sp) == want[:3]


def test_config2_reduced_against_oracle(lj):
    from paper_2111_08824_b200 import configs

    inp = configs.config2(scale=6)
    res, br, _ = lj.ALGORITHMS["grmi-inlj"](inp.r, inp.s, 1, dict(lj.DEFAULT_OPTS, **inp.opts))
    rk, rp = inp.r.numpy()
    sk, sp = inp.s.numpy()
    assert res.checksum == oracle.smj_checksum(rk, rp, sk, sp)
    res_b, _, _ = lj.ALGORITHMS["buffered-grmi-inlj"](inp.r, inp.s, 1, dict(lj.DEFAULT_OPTS, **inp.opts))
    assert res_b.checksum == res.checksum


def test_edge_cases(lj):
    empty = lj.Relation(np.empty(0, np.uint64), np.empty(0, np.uint64))
    one = lj.make_relation(np.array([7], np.uint64), 1)
    for algo in ("grmi-inlj", "buffered-grmi-inlj", "spline-hash-inlj"):
        for r, s in ((empty, one), (one, empty), (one, one)):
            res, _, _ = lj.ALGORITHMS[algo](r, s, 1, dict(lj.DEFAULT_OPTS))
            assert res.checksum == oracle.nlj_checksum(*r.numpy(), *s.numpy()), algo
    # keys at the top of the u64 range, all-duplicate build side
    big = np.array([2**64 - 2, 2**64 - 3, 2**63, 2**63 + 1, 0, 1], np.uint64)
    dup = np.full(50, 12345, np.uint64)
    for keys in (big, dup):
        r = lj.make_relation(keys, 3)
        s = lj.make_relation(np.concatenate([keys, keys[:3], np.array([99], np.uint64)]), 4)
        want = oracle.nlj_checksum(*r.numpy(), *s.numpy())
        for algo in ("grmi-inlj", "buffered-grmi-inlj", "spline-hash-inlj"):
            res, _, _ = lj.ALGORITHMS[algo](r, s, 2, dict(lj.DEFAULT_OPTS, gap_factor=2.5, rmi_fanout=3))
            assert res.checksum == want, (algo, keys[:3])
    with pytest.raises(ValueError):
        lj.Relation(np.array([2**64 - 1], np.uint64), np.array([1], np.uint64))


def test_linearity_over_s_slices(lj):
    """Size-independent property: the checksum of S equals the combination
    of the checksums of its two halves (counts and sums add, xors xor)."""
    from paper_2111_08824_b200 import configs

    inp = configs.config1(scale=2)
    idx = lj.GappedRmiIndex(2.0, 256).fit(inp.r)
    n = len(inp.s)
    a = idx.join_checksum(inp.s.keys[: n // 3], inp.s.payloads[: n // 3]).cpu().tolist()
    b = idx.join_checksum(inp.s.keys[n // 3:], inp.s.payloads[n // 3:]).cpu().tolist()
    w = idx.join_checksum(inp.s.keys, inp.s.payloads).cpu().tolist()
    assert w[0] == a[0] + b[0] and (w[1] - a[1] - b[1]) & MASK == 0 and w[2] == a[2] ^ b[2] and w[3] == a[3] + b[3]


def test_lsj_matches_reference_with_reference_models(golden, lj):
    """lsj.py:373-405 with the reference's own sample models: identical
    checksum AND identical sort counters (comparator_count,
    partitions_sorted); with the GPU's own sample models the checksum is
    unchanged (model neutrality); materialised pairs equal the NLJ oracle."""
    for case, d in golden("lsj").items():
        r = lj.Relation(d["r_keys"], d["r_payloads"])
        s = lj.Relation(d["s_keys"], d["s_payloads"])
        cfg = lj.LsjConfig(workers=int(d["workers"]), fanout=int(d["fanout"]), sample_rate=float(d["sample_rate"]))
        want = tuple(int(v) for v in d["checksum"])
        res, br = lj.lsj_join(r, s, cfg, models=(ref_rmi(lj, d, "mr_"), ref_rmi(lj, d, "ms_")))
        assert res.checksum == want, case
        assert (br.sort_stats.comparator_count, br.sort_stats.partitions_sorted) == tuple(
            int(v) for v in d["sort_stats"]), case
        own, _ = lj.lsj_join(r, s, cfg)
        assert own.checksum == want, case
        mat, _ = lj.lsj_join(r, s, cfg, materialize=True)
        assert mat.checksum == want, case
        assert mat.count == want[0]


def test_lsj_sort_phase_sorted_and_pairs_kept(lj):
    """Global sortedness after the sort phase, pairs still attached
    (tests/test_lsj.py:143-155, 225-232 analogues) on skewed duplicated keys."""
    from paper_2111_08824_b200.lsj import sort_relation

    rng = np.random.default_rng(5)
    base = np.unique(np.floor(2.0**40 * rng.lognormal(0, 1.5, 60000)).astype(np.uint64))
    w = 1.0 / np.arange(1, base.size + 1)
    keys = base[rng.choice(base.size, 200000, p=w / w.sum())]
    pays = np.arange(1, keys.size + 1, dtype=np.uint64)
    r = lj.Relation(keys, pays)
    m = lj.RecursiveModelIndex(100).fit(np.sort(keys[::10]))
    srt = sort_relation(r.keys, r.payloads, m, 64)
    k = _np(srt.keys.contiguous())
    p = _np(srt.payloads.contiguous())
    assert np.all(k[:-1] <= k[1:])
    assert sorted(zip(k.tolist(), p.tolist())) == sorted(zip(keys.tolist(), pays.tolist()))
    bb = srt.bucket_bounds.cpu().numpy()
    part = _i64(lj.partition_index(m, srt.keys.contiguous(), 64))
    assert np.array_equal(np.bincount(part, minlength=64), np.diff(bb))


def test_lsj_edge_cases(lj):
    empty = lj.Relation(np.empty(0, np.uint64), np.empty(0, np.uint64))
    one = lj.make_relation(np.array([7], np.uint64), 1)
    res, _ = lj.lsj_join(empty, one)
    assert res.count == 0
    res, _ = lj.lsj_join(one, one)
    assert res.checksum == oracle.nlj_checksum(*one.numpy(), *one.numpy())
    # duplicate products 2 x 3 = 6 (tests/test_lsj.py:178-182)
    r = lj.make_relation(np.array([7, 7, 9], np.uint64), 1)
    s = lj.make_relation(np.array([7, 7, 7, 8], np.uint64), 2)
    res, _ = lj.lsj_join(r, s, lj.LsjConfig(fanout=50, sample_rate=1.0))
    assert res.count == 6
    # disjoint ranges
    r = lj.make_relation(np.arange(0, 100, dtype=np.uint64), 1)
    s = lj.make_relation(np.arange(1000, 1100, dtype=np.uint64), 2)
    assert lj.lsj_join(r, s, lj.LsjConfig(fanout=50, sample_rate=1.0))[0].count == 0
    # one repeated key larger than shared memory on both sides of the join
    r = lj.make_relation(np.concatenate([np.full(10000, 5, np.uint64), np.arange(10, 20000, dtype=np.uint64)]), 1)
    s = lj.make_relation(np.concatenate([np.full(30000, 5, np.uint64), np.arange(0, 40000, 3, dtype=np.uint64)]), 2)
    res, _ = lj.lsj_join(r, s, lj.LsjConfig(fanout=8, sample_rate=0.05))
    assert res.checksum == oracle.smj_checksum(*r.numpy(), *s.numpy())
    with pytest.raises(lj.ModelMismatchError):
        from paper_2111_08824_b200.lsj import chunked_join, sort_relation

        m1 = lj.RecursiveModelIndex(2).fit(np.arange(100, dtype=np.uint64))
        m2 = lj.RecursiveModelIndex(2).fit(np.arange(100, dtype=np.uint64))
        a = sort_relation(r.keys, r.payloads, m1, 8)
        chunked_join(a, a, m2, 8)


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_lsj_configs_reduced_against_oracle(lj, cfg):
    from paper_2111_08824_b200 import configs

    inp = configs.CONFIGS[cfg](scale=8)
    res, br, _ = lj.ALGORITHMS["lsj"](inp.r, inp.s, 1, dict(lj.DEFAULT_OPTS, **inp.opts))
    assert res.checksum == oracle.smj_checksum(*inp.r.numpy(), *inp.s.numpy())
    assert br.sort_stats.partitions_sorted > 0


def test_config3_reduced_against_oracle(lj):
    from paper_2111_08824_b200 import configs

    inp = configs.config3(scale=64)
    res, _, _ = lj.ALGORITHMS["spline-hash-inlj"](inp.r, inp.s, 1, dict(lj.DEFAULT_OPTS, **inp.opts))
    assert res.checksum == oracle.smj_checksum(*inp.r.numpy(), *inp.s.numpy())
    assert res.count == len(inp.s)  # every probe is an R key, R unique


@pytest.mark.parametrize("fanout", [4, 256, 4096])
def test_buffered_staged_probe_equals_direct(lj, fanout):
    """K4 + staged K1 == K1: identical checksum AND search_steps, including
    searches that leave the staged window (tiny fanout -> long searches)
    and window segments too small to stage."""
    from paper_2111_08824_b200 import configs

    inp = configs.config2(scale=5)
    idx = lj.GappedRmiIndex(2.0, fanout).fit(inp.r)
    direct = idx.join_checksum(inp.s.keys, inp.s.payloads).cpu().tolist()
    buffered = idx.join_checksum_buffered(inp.s.keys, inp.s.payloads).cpu().tolist()
    assert buffered == direct
    small = idx.join_checksum_buffered(inp.s.keys[:5000], inp.s.payloads[:5000]).cpu().tolist()
    assert small == idx.join_checksum(inp.s.keys[:5000], inp.s.payloads[:5000]).cpu().tolist()


def test_buffered_staged_probe_duplicates_and_zero_payloads(lj):
    """Staged K1 on an R with long equal-key runs (some longer than the
    staged halo) and real payloads of 0 (bitmap occupancy): identical to the
    direct probe and to the oracle (checksum and search_steps)."""
    rng = np.random.default_rng(11)
    base = np.unique(rng.integers(0, 2**63, 40000, dtype=np.uint64))
    reps = rng.integers(1, 4, base.size)
    reps[::997] = 3000  # runs that cross window + halo boundaries
    keys = np.repeat(base, reps)
    pays = rng.integers(0, 5, keys.size, dtype=np.uint64)  # many zeros
    r = lj.Relation(keys, pays)
    idx = lj.GappedRmiIndex(2.0, 64).fit(r)
    assert idx.payload_nonzero == 0
    sk = np.concatenate([base[rng.integers(0, base.size, 400000)], rng.integers(0, 2**63, 40000, dtype=np.uint64)])
    sp = rng.integers(0, 2**64 - 1, sk.size, dtype=np.uint64)
    s = lj.Relation(sk, sp)
    direct = idx.join_checksum(s.keys, s.payloads).cpu().tolist()
    buffered = idx.join_checksum_buffered(s.keys, s.payloads).cpu().tolist()
    assert buffered == direct
    # the same through the precomputed staging image
    idx.STAGE_IMAGE_MIN_SLOTS = 0
    idx.__dict__.pop("_stage_img", None)  # drop the cached "no image" decision
    assert idx.stage_image() is not None
    assert idx.join_checksum_buffered(s.keys, s.payloads).cpu().tolist() == direct
    og = oracle.grmi_build(keys, pays, 2.0, 64, model=oracle.Rmi(
        idx.rmi.root_slope, idx.rmi.root_intercept, idx.rmi.trained_len, idx.rmi.leaf_slope, idx.rmi.leaf_intercept,
        idx.rmi.clamp_lo, idx.rmi.clamp_hi, idx.rmi.err_lo, idx.rmi.err_hi))
    want = oracle.grmi_join(og, sk, sp)
    assert (direct[0], direct[1] & MASK, direct[2] & MASK, direct[3]) == want


def test_spline_hash_grouped_probe_equals_direct(lj):
    from paper_2111_08824_b200 import configs

    inp = configs.config3(scale=64)
    idx = lj.SplineHashIndex(32, 18, 4.0).fit(inp.r)
    direct = idx.join_checksum(inp.s.keys, inp.s.payloads).cpu().tolist()
    grouped = idx.join_checksum_buffered(inp.s.keys, inp.s.payloads).cpu().tolist()
    assert grouped == direct
    want = oracle.smj_checksum(*inp.r.numpy(), *inp.s.numpy())
    assert (direct[0], direct[1] & MASK, direct[2] & MASK) == want


def test_partition_fallback_on_unaligned_columns(lj):
    """Key/payload columns that are not 16-B aligned take the plain-load
    partition kernels (no bulk copies); results are unchanged (K4 and LSJ)."""
    from paper_2111_08824_b200 import configs

    inp = configs.config2(scale=6)
    idx = lj.GappedRmiIndex(2.0, 1024).fit(inp.r)
    n = len(inp.s) - 1
    base = idx.join_checksum(inp.s.keys[1:], inp.s.payloads[1:]).cpu().tolist()
    k1, p1 = inp.s.keys[1:], inp.s.payloads[1:]  # 8-B aligned views
    assert k1.data_ptr() % 16 == 8
    got = idx.join_checksum_buffered(k1, p1).cpu().tolist()
    assert got == base
    # LSJ on unaligned views of both relations
    r = lj.Relation(inp.r.keys[1:].contiguous(), inp.r.payloads[1:].contiguous())
    s = lj.Relation(inp.s.keys[1:n // 2], inp.s.payloads[1:n // 2], validate=False)
    assert s.keys.data_ptr() % 16 == 8
    res, _ = lj.lsj_join(r, s)
    assert res.checksum == oracle.smj_checksum(*r.numpy(), *s.numpy())


def test_rmi_inlj_bitwise_with_reference_model(golden, lj):
    """K12 rmi-inlj (baselines.py:96-157) over the reference's sorted R and
    fitted model: the reference's checksum and search_steps."""
    import torch

    from paper_2111_08824_b200.joins import rmi_inlj

    for case, d in golden("algos").items():
        order = np.argsort(d["r_keys"], kind="stable")
        rk = torch.from_numpy(d["r_keys"][order].view(np.int64)).cuda()
        rp = torch.from_numpy(d["r_payloads"][order].view(np.int64)).cuda()
        s = lj.Relation(d["s_keys"], d["s_payloads"])
        for w in (1, 4):
            words = rmi_inlj(rk, rp, ref_rmi(lj, d, "rmi_"), s, w).cpu().tolist()
            assert (words[0], words[1] & MASK, words[2] & MASK) == tuple(int(v) for v in d["checksum"]), case
            assert words[3] == int(d[f"rmi-inlj_w{w}_counters"][0]), (case, w)


def test_key_file_roundtrip_to_device_and_canonical(lj, tmp_path):
    """data.py:195-216 key files loaded straight to the
    device bit-exactly (corrupt headers rejected), and JoinResult.canonical
    computed on the device equals the reference's np.lexsort order."""
    rng = np.random.default_rng(9)
    keys = np.concatenate([rng.integers(0, 2**63, 5000, dtype=np.uint64), np.array([0, 2**63 - 1], np.uint64)])
    path = tmp_path / "k.bin"
    lj.write_keys_file(path, keys)
    dev = lj.load_keys_file(path)
    assert dev.is_cuda and np.array_equal(_np(dev), keys)
    bad = tmp_path / "bad.bin"
    bad.write_bytes(path.read_bytes()[:-8])
    with pytest.raises(lj.CorruptKeyFileError):
        lj.load_keys_file(bad)
    r = lj.relation_from_keys_file(path, 5)
    assert np.array_equal(r.numpy()[1], lj.make_relation(keys, 5).numpy()[1])
    s = lj.make_relation(np.concatenate([keys[:300], keys[:100]]), 6)
    res, _, _ = lj.ALGORITHMS["grmi-inlj"](r, s, 1, dict(lj.DEFAULT_OPTS, materialize=True))
    pr, ps = res.payloads_r, res.payloads_s
    order = np.lexsort((ps, pr))
    want = np.column_stack((pr[order], ps[order]))
    assert np.array_equal(res.canonical(), want)
    dr, ds = res.canonical_device()
    assert np.array_equal(np.column_stack((_np(dr), _np(ds))), want)


# ---- the key-range bin structure (lj_keybin.cuh) the partition passes use


def _keybin(bounds, keys):
    from paper_2111_08824_b200 import _lib

    lib = _lib.lib()
    nb = len(bounds)
    b = torch.from_numpy(np.ascontiguousarray(bounds, np.uint64).view(np.int64)).cuda()
    k = torch.from_numpy(np.ascontiguousarray(keys, np.uint64).view(np.int64)).cuda()
    out = torch.empty(max(len(keys), 1), dtype=torch.int32, device="cuda")
    ws = _lib.workspace(lib.lj_keybin_workspace_bytes(nb))
    _lib.check(lib.lj_keybin_eval(_lib.ptr(b), nb, _lib.ptr(k), len(keys), _lib.ptr(out), _lib.ptr(ws), ws.numel(),
                                  _lib.stream_ptr()), "keybin_eval")
    return out[: len(keys)].cpu().numpy().astype(np.int64)


def _dist_keys(rng, dist, n):
    if dist == "uniform":
        return rng.integers(0, 2**63, n, dtype=np.uint64)
    if dist == "lognormal":
        return np.floor(1e12 * rng.lognormal(0, 2, n)).astype(np.uint64)
    if dist == "clusters":
        c = rng.integers(0, 2**62, 64).astype(np.float64)
        return np.clip(c[rng.integers(0, 64, n)] + rng.normal(0, 2.0**40, n), 0, 2.0**63 - 4096).astype(np.uint64)
    if dist == "dups":
        return rng.integers(0, 50, n, dtype=np.uint64) * np.uint64(1 << 40)
    if dist == "dense":
        return rng.integers(10**6, 10**6 + 5000, n, dtype=np.uint64)
    return np.uint64(2**64 - 2) - rng.integers(0, 10**6, n, dtype=np.uint64)  # "top" of the key space


@pytest.mark.parametrize("dist", ["uniform", "lognormal", "clusters", "dups", "dense", "top"])
@pytest.mark.parametrize("nb", [1, 2, 37, 512, 1000, 2048])
def test_keybin_matches_search(lj, dist, nb):
    """bin(k) = #{ j >= 1 : B[j] <= k } exactly, whichever key image the
    table picks, on boundaries drawn from the distribution (repeats and all)
    and keys on, next to and between them."""
    rng = np.random.default_rng(nb * 7 + len(dist))
    bounds = np.sort(_dist_keys(rng, dist, nb))
    bounds[0] = 0
    inner = bounds[1:]
    keys = np.concatenate([_dist_keys(rng, dist, 20000), inner, inner - np.minimum(inner, 1),
                           np.minimum(inner, np.uint64(2**64 - 3)) + np.uint64(1),
                           np.array([0, 1, 2**63 - 1, 2**63, 2**64 - 2], dtype=np.uint64)])
    want = np.searchsorted(inner, keys, side="right")
    assert np.array_equal(_keybin(bounds, keys), want)


@pytest.mark.parametrize("dist", ["uniform", "lognormal", "clusters", "dense"])
def test_lsj_key_bounds_equal_model_bins(lj, dist):
    """The partition's key-range bins are the model's bins table[pos(key)]
    on every key (sample keys, draws, boundaries and their neighbours)."""
    from paper_2111_08824_b200 import _lib, lsj

    rng = np.random.default_rng(11)
    rk = np.unique(_dist_keys(rng, dist, 300000))
    r = lj.make_relation(rk, 3)
    _, lm = lsj.prepare_model(r, 0.01, 5)
    lib = _lib.lib()
    bounds = torch.empty(lm.nbins, dtype=torch.int64, device="cuda")
    ws = _lib.workspace(lib.lj_keybin_workspace_bytes(lm.nbins))
    c = lm.c_struct()
    _lib.check(lib.lj_lsj_key_bounds(ctypes.byref(c), _lib.ptr(bounds), _lib.ptr(ws), ws.numel(), _lib.stream_ptr()),
               "lsj_key_bounds")
    b = _np(bounds)
    inner = b[1:]
    keys = np.concatenate([rk, _dist_keys(rng, dist, 50000), inner, inner - np.minimum(inner, 1),
                           np.array([0, 1, 2**63 - 1], dtype=np.uint64)])
    pos = lm.rmi.predict_many(keys)[0]
    model_bins = lm.table.long()[pos].cpu().numpy()
    assert np.array_equal(_keybin(b, keys), model_bins)


@pytest.mark.parametrize("buffered", [True, False])
def test_join_checksum_host_streams_chunks(lj, buffered):
    """Host-resident S streamed in chunks (copies overlapped with the join)
    gives the same words as the device-resident join; the reserved key is
    rejected."""
    rng = np.random.default_rng(21)
    rk = np.unique(rng.integers(0, 2**63, 50000, dtype=np.uint64))
    sk = np.concatenate([rng.choice(rk, 90000), rng.integers(0, 2**63, 7000, dtype=np.uint64)])
    r = lj.make_relation(rk, 1)
    s = lj.make_relation(sk, 2)
    hk, hp = s.keys.cpu(), s.payloads.cpu()
    for idx in (lj.GappedRmiIndex(2.0, 256).fit(r), lj.SplineHashIndex(32, 18, 4.0).fit(r)):
        want = idx.join_checksum(s.keys, s.payloads).cpu().tolist()
        for chunk in (1000, 33333, 1 << 20):
            got = lj.join_checksum_host(idx, hk, hp, buffered=buffered, chunk=chunk).cpu().tolist()
            assert got == want, (type(idx).__name__, chunk)
    bad = hk.clone()
    bad[500] = -1
    with pytest.raises(ValueError):
        lj.join_checksum_host(idx, bad, hp, buffered=buffered, chunk=1000)


@pytest.mark.parametrize("shuffle", ["fused", "nccl"])
def test_distributed_lsj_single_rank_nccl(lj, tmp_path, monkeypatch, shuffle):
    """The C5 path (shared model, range shuffle -- fused partition + P2P
    stores into symmetric memory, or partition + NCCL all-to-all-v -- local
    LSJ, 3-word reduction) on a one-rank NCCL group equals the oracle; the
    exchange protocol at world 2 is covered with gloo in test_dist.py."""
    monkeypatch.setenv("LJ_SHUFFLE", shuffle)
    import torch.distributed as dist

    from paper_2111_08824_b200 import configs
    from paper_2111_08824_b200 import dist as ljdist

    inp = configs.config5(scale=12)
    want = oracle.smj_checksum(*inp.r.numpy(), *inp.s.numpy())
    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        (c, s, x), ph = ljdist.lsj_join(inp.r.keys, inp.r.payloads, inp.s.keys, inp.s.payloads,
                                        lj.LsjConfig(fanout=4096, sample_rate=0.01))
        ljdist._SYMM.clear()
    finally:
        dist.destroy_process_group()
    assert (c, s, x) == tuple(want)
    assert ph["shuffle"] == ("fused P2P" if shuffle == "fused" else "partition + NCCL all-to-all-v")


def test_lsj_on_shuffled_orders_repeatedly(lj):
    """The local LSJ of the distributed path sees its relations in the
    nondeterministic order of the claims scatter; some orders (the sample
    then fits a model whose last leaf leaves the top keys' placement
    misordered) need the sort's sortedness check + whole-bucket fallback.
    Dropping that check broke ~1 in 8 of these runs (a C5 shard); 24 runs
    over scatter-ordered relations must all be exact."""
    from paper_2111_08824_b200 import configs
    from paper_2111_08824_b200.lsj import LsjModel, _partition
    from paper_2111_08824_b200.models import RecursiveModelIndex

    inp = configs.config5(scale=12)
    want = tuple(oracle.smj_checksum(*inp.r.numpy(), *inp.s.numpy()))
    cfg = lj.LsjConfig(fanout=4096, sample_rate=0.01)
    # a one-bin partition is a claims scatter: a nondeterministic permutation
    from paper_2111_08824_b200.util import sort_pairs
    srt, _ = sort_pairs(inp.r.keys[::64].contiguous(), inp.r.keys[::64].contiguous())
    one = LsjModel.from_sample(RecursiveModelIndex(16).fit(srt), srt, 1)
    for rep in range(24):
        pr, _ = _partition(inp.r.keys, inp.r.payloads, one)
        ps, _ = _partition(inp.s.keys, inp.s.payloads, one)
        pr, ps = pr.view(-1, 2), ps.view(-1, 2)
        r = lj.Relation(pr[:, 0].contiguous(), pr[:, 1].contiguous(), validate=False)
        s = lj.Relation(ps[:, 0].contiguous(), ps[:, 1].contiguous(), validate=False)
        res, br = lj.lsj_join(r, s, cfg)
        assert res.checksum == want, rep
        # placement is monotone (keys past the training range sort at the
        # top): the whole-bucket fallback never has to fire
        assert br.extra["r_bitonic_fallbacks"] == 0 and br.extra["s_bitonic_fallbacks"] == 0, rep


def test_lsj_join_host_overlapped_equals_device(lj):
    """lsj_join_host (R's side overlapped with S's H2D) == lsj_join == oracle."""
    from paper_2111_08824_b200 import configs

    inp = configs.config4(scale=10)
    cfg = lj.LsjConfig(fanout=4096, sample_rate=0.01)
    want, _ = lj.lsj_join(inp.r, inp.s, cfg)
    got = lj.lsj_join_host(inp.r.keys.cpu(), inp.r.payloads.cpu(), inp.s.keys.cpu(), inp.s.payloads.cpu(), cfg)
    assert got.checksum == want.checksum == tuple(oracle.smj_checksum(*inp.r.numpy(), *inp.s.numpy()))


def test_lsj_join_wide_r_slices(lj):
    """A sparse S against a dense R: every S tile faces an R slice far wider
    than one shared-memory chunk (and equal-key runs of R that cross chunk
    boundaries): the chunked merge equals the oracle."""
    rng = np.random.default_rng(23)
    base = np.unique(rng.integers(0, 2**40, 400000, dtype=np.uint64))
    reps = np.ones(base.size, dtype=np.int64)
    reps[::50000] = 9000  # runs longer than a chunk
    rk = np.repeat(base, reps)
    sk = np.concatenate([rng.choice(base, 3000), base[::50000], rng.integers(0, 2**40, 500, dtype=np.uint64)])
    r = lj.make_relation(rk, 5)
    s = lj.make_relation(sk, 6)
    for fanout in (64, 4096):
        res, _ = lj.lsj_join(r, s, lj.LsjConfig(fanout=fanout, sample_rate=0.05))
        assert res.checksum == tuple(oracle.smj_checksum(*r.numpy(), *s.numpy())), fanout


def _fit_both(lj, keys, err=32, bits=18, monkeypatch=None):
    k = np.sort(np.asarray(keys, dtype=np.uint64))
    dev = torch.from_numpy(k.view(np.int64)).cuda()
    gpu = lj.RadixSplineIndex(err, bits).fit(dev)
    monkeypatch.setenv("LJ_HOST_SPLINE_FIT", "1")
    host = lj.RadixSplineIndex(err, bits).fit(dev)
    monkeypatch.delenv("LJ_HOST_SPLINE_FIT")
    return gpu, host


@pytest.mark.parametrize("dist", ["uniform", "lognormal", "clusters", "dups", "dense", "linear", "collide53"])
def test_spline_fit_on_device_equals_host(lj, dist, monkeypatch):
    """The device greedy corridor (speculative chunks spliced where they
    converge, repaired in order where they do not) gives the host fit's --
    the reference's -- knots, ranks, radix table and shift exactly.
    "linear" has chunks without any knot (the repair path); "collide53" has
    distinct keys that round to the same float64."""
    rng = np.random.default_rng(31)
    n = 300_000
    if dist == "linear":
        keys = np.arange(n, dtype=np.uint64) * np.uint64(7919) + np.uint64(10**9)
    elif dist == "collide53":
        keys = np.uint64(2**60) + rng.integers(0, 2**12, n, dtype=np.uint64) * np.uint64(3)
    else:
        keys = _dist_keys(rng, dist, n)
    for err, bits in ((32, 18), (4, 10), (1, 20)):
        gpu, host = _fit_both(lj, keys, err, bits, monkeypatch)
        assert np.array_equal(gpu.spline_keys, host.spline_keys), (dist, err)
        assert np.array_equal(gpu.spline_ranks, host.spline_ranks), (dist, err)
        assert np.array_equal(gpu.radix_table, host.radix_table), (dist, err)
        assert int(gpu.shift) == int(host.shift)


def test_spline_fit_on_device_matches_golden(golden, lj, monkeypatch):
    """The reference-fitted splines of the golden vectors, refit on device."""
    checked = 0
    for name, d in golden("models").items():
        if "sp_keys" not in d:
            continue
        k = np.sort(np.asarray(d["keys"], dtype=np.uint64))
        dev = torch.from_numpy(k.view(np.int64)).cuda()
        m = lj.RadixSplineIndex(int(d["sp_max_error"]), int(d["sp_radix_bits"])).fit(dev)
        assert np.array_equal(m.spline_keys, np.asarray(d["sp_keys"], dtype=np.uint64)), name
        assert np.array_equal(m.spline_ranks, np.asarray(d["sp_ranks"], dtype=np.int64)), name
        assert np.array_equal(m.radix_table, np.asarray(d["sp_radix_table"], dtype=np.int64)), name
        assert int(m.shift) == int(d["sp_shift"]), name
        checked += 1
    assert checked >= 5


@pytest.mark.parametrize("keys", [[5], [5, 9], [5, 9, 11], [7] * 1000, [3] * 500 + [8] * 500,
                                  [0, 2**63 - 1], list(range(70000))])
def test_spline_fit_on_device_small_and_degenerate(lj, keys, monkeypatch):
    """Device fit == host fit on one, two and three points, all-equal keys,
    two distinct keys, the extremes of the key domain and a knot-free line
    longer than two chunks."""
    gpu, host = _fit_both(lj, keys, 32, 18, monkeypatch)
    assert np.array_equal(gpu.spline_keys, host.spline_keys)
    assert np.array_equal(gpu.spline_ranks, host.spline_ranks)
    assert np.array_equal(gpu.radix_table, host.radix_table)
    assert int(gpu.shift) == int(host.shift)


def test_host_resident_entry_points_on_empty_inputs(lj):
    r = lj.make_relation(np.arange(100, dtype=np.uint64) * 3, 1)
    e = torch.empty(0, dtype=torch.int64)
    idx = lj.GappedRmiIndex(2.0, 16).fit(r)
    assert lj.join_checksum_host(idx, e, e).cpu().tolist() == [0, 0, 0, 0]
    res = lj.lsj_join_host(r.keys.cpu(), r.payloads.cpu(), e, e)
    assert res.checksum == (0, 0, 0)


def _dup_probe_sets():
    rng = np.random.default_rng(31)
    base = np.unique(rng.integers(0, 2**40, 50000, dtype=np.uint64))
    dup = np.concatenate([base, base[::7], base[::7], base[::101]])  # equal build keys: adjacent real slots
    clus = np.unique(np.concatenate([rng.normal(c, 2**24, 20000) for c in (2**50, 2**51, 3 * 2**52)]).astype(np.uint64))
    high = np.unique(rng.integers(2**63, 2**64 - 1, 30000, dtype=np.uint64))  # keys >= 2^63
    return {"dup": dup, "clusters": clus, "high": high, "tiny1": np.array([5], np.uint64),
            "tiny3": np.array([9, 9, 2**62], np.uint64)}


@pytest.mark.parametrize("name", ["dup", "clusters", "high", "tiny1", "tiny3"])
def test_spline_hash_probe_table_equals_chains(lj, name):
    """The staged probe over the slot table (k_hash_probe_staged) against
    the chain probe (K5) and the oracle: duplicate build keys, clustered
    keys, keys >= 2^63, probes below / above / between the build keys."""
    rk = _dup_probe_sets()[name]
    rng = np.random.default_rng(5)
    sk = np.concatenate([rng.choice(rk, 200000), rng.integers(0, 2**64 - 1, 20000, dtype=np.uint64),
                         np.array([0, rk.min(), rk.max(), 2**64 - 2], np.uint64)])
    sk = rng.permutation(sk)
    r = lj.make_relation(rng.permutation(rk), 3)
    s = lj.make_relation(sk, 4)
    idx = lj.SplineHashIndex(32, 18, 4.0).fit(r)
    assert idx.slots is not None
    want = oracle.smj_checksum(*r.numpy(), *s.numpy())
    direct = idx.join_checksum(s.keys, s.payloads).cpu().tolist()
    grouped = idx.join_checksum_buffered(s.keys, s.payloads).cpu().tolist()
    assert (direct[0], direct[1] & MASK, direct[2] & MASK) == want
    assert (grouped[0], grouped[1] & MASK, grouped[2] & MASK) == want


def test_spline_hash_zero_payloads_keep_the_chains(lj):
    rk = np.unique(np.random.default_rng(2).integers(0, 2**50, 40000, dtype=np.uint64))
    rp = np.arange(rk.size, dtype=np.uint64)  # payload 0 once: no gap marker, no slot table
    r = lj.Relation(rk, rp)
    s = lj.make_relation(np.concatenate([rk, rk[:1000]]), 8)
    idx = lj.SplineHashIndex(32, 18, 4.0).fit(r)
    assert idx.slots is None
    want = oracle.smj_checksum(*r.numpy(), *s.numpy())
    g = idx.join_checksum_buffered(s.keys, s.payloads).cpu().tolist()
    assert (g[0], g[1] & MASK, g[2] & MASK) == want


@pytest.mark.parametrize("n", [2000, 9000, 50000])
def test_lsj_sort_flat_model_big_and_global_paths(lj, n):
    """A flat model (fitted on one key: slope 0, every y equal) puts every
    key of a relation into one mixed slice: n = 9000 goes to the big sort
    instance (one CTA per SM), n = 50000 to the global-memory chunk sort +
    merge (k_lsj_huge) -- all device-driven, no host readback.  Sorted,
    pairs kept, and the counters say which path ran."""
    from paper_2111_08824_b200.lsj import LsjModel, sort_diag, sort_relation

    rng = np.random.default_rng(n)
    keys = rng.integers(0, 2**63, n, dtype=np.uint64)
    keys[: n // 10] = keys[n // 10]  # duplicates inside the slice
    pays = rng.integers(1, 2**63, n, dtype=np.uint64)
    r = lj.Relation(keys, pays)
    rmi = lj.RecursiveModelIndex(1).fit(np.array([12345], np.uint64))
    srt = sort_relation(r.keys, r.payloads, LsjModel.uniform(rmi, 1), 1)
    k = _np(srt.keys.contiguous())
    p = _np(srt.payloads.contiguous())
    assert np.all(k[:-1] <= k[1:])
    assert sorted(zip(k.tolist(), p.tolist())) == sorted(zip(keys.tolist(), pays.tolist()))
    d = sort_diag(srt.diag)
    if n > 3072:
        assert d["oversized_sub_buckets"] >= 1
    if n > 12288:
        assert d["global_sorted_sub_buckets"] >= 1


def _lsj_sets():
    from paper_2111_08824_b200 import configs

    rng = np.random.default_rng(17)
    c4 = configs.config4(scale=8)
    c5 = configs.config5(scale=12)
    tiny_r = np.array([3, 9, 9, 2**63 + 1, 40], np.uint64)
    tiny_s = np.array([9, 40, 41, 2**63 + 1, 2**63 + 1, 3], np.uint64)
    zr = np.unique(rng.integers(0, 2**44, 100000, dtype=np.uint64))
    zs = zr[np.minimum(rng.zipf(1.3, 300000), zr.size) - 1]
    return {"c4": (c4.r, c4.s), "c5": (c5.r, c5.s),
            "tiny": (lj_mod().make_relation(tiny_r, 1), lj_mod().make_relation(tiny_s, 2)),
            "zipf": (lj_mod().make_relation(zr, 3), lj_mod().make_relation(zs, 4))}


def lj_mod():
    import paper_2111_08824_b200 as lj

    return lj


@pytest.mark.parametrize("name", ["c4", "c5", "tiny", "zipf"])
def test_lsj_run_one_call_abi_equals_lsj_join_and_oracle(lj, name):
    """lj_lsj_run (the whole LSJ in one asynchronous C call, one workspace)
    through ctypes == lsj_join (Python orchestration) == the oracle."""
    r, s = _lsj_sets()[name]
    want = oracle.smj_checksum(*r.numpy(), *s.numpy())
    cfg = lj.LsjConfig(fanout=4096, sample_rate=0.01)
    got = lj.lsj_run(r, s, cfg).checksum
    res, _ = lj.lsj_join(r, s, cfg)
    assert got == tuple(want) == res.checksum


@pytest.mark.parametrize("name", ["c4", "zipf"])
def test_lsj_one_pass_partition_equals_exact_and_overflow_falls_back(lj, name, monkeypatch):
    """LSJ's partition in ONE pass (sample-sized regions with gaps,
    lj_lsj_partition_regions + lj_lsj_sort_regions) == the exact two-pass
    partition == the oracle; with the regions' slack taken away
    (LJ_EST_TIGHT: about half of the bins overflow) the device-side
    fallback to the exact partition gives the same join, through both the
    Python orchestration and the one-call ABI."""
    r, s = _lsj_sets()[name]
    want = tuple(oracle.smj_checksum(*r.numpy(), *s.numpy()))
    cfg = lj.LsjConfig(fanout=4096, sample_rate=0.01)
    res, br = lj.lsj_join(r, s, cfg)
    assert res.checksum == want
    monkeypatch.setenv("LJ_LSJ_EXACT_PARTITION", "1")
    exact, br2 = lj.lsj_join(r, s, cfg)
    assert exact.checksum == want
    assert br.sort_stats == br2.sort_stats  # the reference counters: the same sorted relations
    monkeypatch.delenv("LJ_LSJ_EXACT_PARTITION")
    monkeypatch.setenv("LJ_EST_TIGHT", "1")
    tight, br3 = lj.lsj_join(r, s, cfg)
    assert tight.checksum == want
    assert br3.sort_stats == br2.sort_stats
    assert lj.lsj_run(r, s, cfg).checksum == want


@pytest.mark.parametrize("name", ["c4", "zipf", "tiny", "c5"])
def test_lsj_from_interleaved_records_equals_columns_and_oracle(lj, name, monkeypatch):
    """A RecordRelation (interleaved 16-B records, the distributed LSJ's
    receive buffer) is sampled and partitioned in place
    (lj_lsj_sample_strided, lj_lsj_partition_regions_rec): every bin holds
    the same multiset as the column partition's, the join equals the column
    join and the oracle -- also through the overflow fallback (LJ_EST_TIGHT)
    and with the exact partition forced (records copied to columns)."""
    r, s = _lsj_sets()[name]
    want = tuple(oracle.smj_checksum(*r.numpy(), *s.numpy()))
    cfg = lj.LsjConfig(fanout=4096, sample_rate=0.01)
    rr = lj.RecordRelation(torch.stack([r.keys, r.payloads], dim=1))
    sr = lj.RecordRelation(torch.stack([s.keys, s.payloads], dim=1))
    assert torch.equal(rr.keys, r.keys) and torch.equal(sr.payloads, s.payloads)
    from paper_2111_08824_b200 import lsj as L

    _, lm = L.prepare_model(r, cfg.sample_rate, cfg.seed)
    _, lm2 = L.prepare_model(rr, cfg.sample_rate, cfg.seed)
    assert torch.equal(lm.pb, lm2.pb)  # the strided sample draws the same keys
    pc, regc = L._partition_regions(r.keys, r.payloads, lm)
    pr, regr = L._partition_regions_rec(rr.records, lm)
    assert torch.equal(regc, regr)
    nb = lm.nbins
    reg = regc.cpu().tolist()
    for b in sorted({0, min(1, nb - 1), nb // 2, nb - 1}):
        a, e = reg[b], reg[nb + 1 + b]
        kc, kr = pc[2 * a:2 * e:2], pr[2 * a:2 * e:2]
        oc, orr = torch.argsort(kc), torch.argsort(kr)
        assert torch.equal(kc[oc], kr[orr])
        assert torch.equal(pc[2 * a + 1:2 * e:2][oc].sort().values, pr[2 * a + 1:2 * e:2][orr].sort().values)
    res, br = lj.lsj_join(rr, sr, cfg)
    ref, br0 = lj.lsj_join(r, s, cfg)
    assert res.checksum == want == ref.checksum
    assert br.sort_stats == br0.sort_stats
    mixed, _ = lj.lsj_join(r, sr, cfg)  # one side as records
    assert mixed.checksum == want
    assert lj.lsj_run(rr, sr, cfg).checksum == want  # lj_lsj_run_rec: the one-call ABI over records
    assert lj.lsj_run(rr, s, cfg).checksum == want
    monkeypatch.setenv("LJ_EST_TIGHT", "1")
    assert lj.lsj_join(rr, sr, cfg)[0].checksum == want
    monkeypatch.delenv("LJ_EST_TIGHT")
    monkeypatch.setenv("LJ_LSJ_EXACT_PARTITION", "1")
    assert lj.lsj_join(rr, sr, cfg)[0].checksum == want


def test_record_relation_edge_cases(lj):
    """Odd sizes (tiles with a tail), tiny relations (the zero-sample
    fallback) and an empty side through the record path."""
    g = torch.Generator(device="cuda").manual_seed(5)
    for n in (1, 2, 7, 4097, 100003):
        k = torch.randperm(4 * n, generator=g, device="cuda")[:n].to(torch.int64) * 977 + 13
        p = k * 3 + 1
        sk = k[torch.randint(0, n, (2 * n + 1,), generator=g, device="cuda")]
        sp = sk ^ 0x55
        want = tuple(oracle.smj_checksum(k.cpu().numpy().view("u8"), p.cpu().numpy().view("u8"),
                                         sk.cpu().numpy().view("u8"), sp.cpu().numpy().view("u8")))
        rr = lj.RecordRelation(torch.stack([k, p], dim=1))
        sr = lj.RecordRelation(torch.stack([sk, sp], dim=1))
        assert lj.lsj_join(rr, sr, lj.LsjConfig(sample_rate=0.01))[0].checksum == want
        assert lj.lsj_run(rr, sr, lj.LsjConfig(sample_rate=0.01)).checksum == want
    empty = lj.RecordRelation(torch.empty((0, 2), dtype=torch.int64, device="cuda"))
    assert lj.lsj_join(empty, sr)[0].checksum == (0, 0, 0)
    with pytest.raises(ValueError):
        lj.RecordRelation(torch.zeros(4, dtype=torch.int64, device="cuda"))


def test_lsj_run_replays_as_a_cuda_graph(lj):
    """lj_lsj_run enqueues everything on the stream (no host readback, the
    partition's overflow fallback decided on the device), so the whole
    learned sort-join captures into ONE CUDA graph; replays on fresh
    result words equal the oracle."""
    r, s = _lsj_sets()["c4"]
    want = tuple(oracle.smj_checksum(*r.numpy(), *s.numpy()))
    cfg = lj.LsjConfig(fanout=4096, sample_rate=0.01)
    assert lj.lsj_run(r, s, cfg).checksum == want  # warm-up: kernel attributes are set outside the capture
    from paper_2111_08824_b200 import _lib

    lib = _lib.lib()
    dev = r.keys.device
    out = torch.zeros(4, dtype=torch.int64, device=dev)
    ws = _lib.workspace(lib.lj_lsj_run_workspace_bytes(len(r), len(s), float(cfg.sample_rate)), dev)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            _lib.check(lib.lj_lsj_run(_lib.ptr(r.keys), _lib.ptr(r.payloads), len(r), _lib.ptr(s.keys),
                                      _lib.ptr(s.payloads), len(s), float(cfg.sample_rate),
                                      int(cfg.seed) & (2**64 - 1), _lib.ptr(out), _lib.ptr(ws), ws.numel(),
                                      _lib.stream_ptr()), "lsj_run")
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert tuple(int(v) & MASK for v in out.cpu().tolist()[:3]) == want


C01_ALGOS = ["grmi-inlj", "buffered-grmi-inlj", "spline-hash-inlj", "lsj", "rmi-inlj"]


@pytest.mark.parametrize("algo", C01_ALGOS)
def test_c01_registry_checksums_and_counters(golden, lj, algo):
    """The reference's acceptance criterion c01 sweep (kinds x n in {1e3,
    1e4} x dup in {0, 0.25, 0.5}, plus n = 1e5 at dup 0.5) through the GPU
    registry at workers 1 and 4: every checksum equals the reference's NLJ
    truth, and the runners' counters equal the reference runners' --
    search_steps / predictions / leaf_switches (the buffered runner's
    flush schedule) for the INLJs, and comparator_count /
    partitions_sorted for LSJ with the reference's sampler."""
    for case, d in golden("c01").items():
        r = lj.Relation(d["r_keys"], d["r_payloads"])
        s = lj.Relation(d["s_keys"], d["s_payloads"])
        for workers in (1, 4):
            opts = dict(lj.DEFAULT_OPTS, lsj_sampler="reference")
            res, br, _ = lj.ALGORITHMS[algo](r, s, workers, opts)
            assert res.checksum == tuple(int(v) for v in d["checksum"]), (case, algo, workers)
            want = [int(v) for v in d[f"{algo}_w{workers}_counters"]]
            c = br.counters()
            got = [c["search_steps"], c["predictions"], c["leaf_switches"], c["comparator_count"],
                   c["partitions_sorted"]]
            if algo == "rmi-inlj":  # steps depend on the fitted model's last bits: the fixture's own model is
                got[0] = want[0] = 0  # pinned in test_rmi_inlj_bitwise_with_reference_model
            assert got == want, (case, algo, workers, got, want)
