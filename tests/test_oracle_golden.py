"""Pin the C oracle (oracle/lj_oracle.c) to golden vectors produced by the
reference package itself (oracle/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle
from conftest import rmi_from_fixture, spline_from_fixture


def test_mix64_and_payloads(golden):
    g = golden("util")
    assert np.array_equal(oracle.mix64(g["x"]), g["mix64"])
    for seed in (0, 1, 42, 2**40 + 5):
        assert np.array_equal(oracle.make_payloads(1000, seed), g[f"payloads_{seed}"])


def test_chunk_bounds(golden):
    for row in golden("util")["chunk_bounds"]:
        n, w = int(row[0]), int(row[1])
        assert np.array_equal(oracle.chunk_bounds(n, w), row[2 : 3 + w])


MODEL_SETS = ["unif63", "lognorm1e12", "clusters", "seq_h", "lognorm_ref", "dups", "linear",
              "tiny", "single", "dbl_collide"]


@pytest.mark.parametrize("name", MODEL_SETS)
def test_rmi_predict_bitwise_with_reference_params(golden, name):
    """models.py:112-135 evaluated by the oracle on the reference-fitted
    parameters is bit-identical to the reference's predict_many."""
    d = golden("models")[name]
    m = rmi_from_fixture(d)
    pos, lo, hi, leaf = oracle.rmi_predict(m, d["probes"])
    assert np.array_equal(pos, d["pos"])
    assert np.array_equal(lo, d["lo"])
    assert np.array_equal(hi, d["hi"])
    assert np.array_equal(leaf, d["route"])
    for P in (1, 7, 4096):
        assert np.array_equal(oracle.rmi_partition_index(m, d["probes"], P), d[f"part_{P}"])


@pytest.mark.parametrize("name", MODEL_SETS)
def test_rmi_fit_matches_reference(golden, name):
    """The oracle's fit differs from numpy only in summation order: integer
    parameters (clamps) match exactly, floats to ~1e-9 relative, and the
    bounds are sound (tests/test_models.py:65-72)."""
    d = golden("models")[name]
    keys = d["keys"]
    m = oracle.rmi_fit(keys, int(d["fanout"]))
    if name != "dbl_collide":
        # (dbl_collide: 3000 keys within 4096 of 2^60, where the root's
        # mean-centring cancels catastrophically and any summation order
        # gives a different, equally sound, root)
        assert np.array_equal(m.clamp_lo, d["clamp_lo"])
        assert np.array_equal(m.clamp_hi, d["clamp_hi"])
        np.testing.assert_allclose(m.leaf_slope, d["leaf_slope"], rtol=1e-6, atol=1e-12)
    pos, lo, hi, _ = oracle.rmi_predict(m, keys)
    truth = np.searchsorted(keys, keys, side="left")
    assert np.all((lo <= truth) & (truth <= hi))
    assert np.all(np.diff(pos) >= 0)


@pytest.mark.parametrize("name", MODEL_SETS)
def test_spline_fit_and_predict_bitwise(golden, name):
    """models.py:171-282: the greedy corridor restated in C chooses exactly
    the reference's spline points; predictions are bit-identical."""
    d = golden("models")[name]
    keys = d["keys"]
    me, rb = int(d["sp_max_error"]), int(d["sp_radix_bits"])
    sp = oracle.spline_fit(keys, me, rb)
    assert np.array_equal(sp.spline_keys, d["sp_keys"])
    assert np.array_equal(sp.spline_ranks, d["sp_ranks"])
    assert np.array_equal(sp.radix_table, d["sp_radix_table"])
    assert sp.shift == int(d["sp_shift"])
    pos, lo, hi = oracle.spline_predict(sp, d["probes"])
    assert np.array_equal(pos, d["sp_pos"])
    assert np.array_equal(lo, d["sp_lo"])
    assert np.array_equal(hi, d["sp_hi"])
    assert np.array_equal(oracle.spline_partition_index(sp, d["probes"], 4 * keys.size), d["sp_part_4n"])
    assert np.array_equal(oracle.spline_partition_index(sp, d["probes"], 3), d["sp_part_3"])


def _grmi_cases(golden):
    return sorted(golden("grmi").keys())


def test_grmi_layout_search_and_join(golden):
    """gapped.py:221-338 with the reference's model: identical gapped arrays,
    predicted slots, per-probe search results and probe counts, run lengths,
    and the join checksum."""
    g = golden("grmi")
    assert len(g) >= 20
    for case, d in g.items():
        m = rmi_from_fixture(d)
        idx = oracle.grmi_build(d["keys"], d["payloads"], float(d["gap"]), int(d["fanout"]), model=m)
        assert idx.L == int(d["L"]), case
        assert np.array_equal(idx.gkeys, d["gkeys"]), case
        assert np.array_equal(idx.gpayloads, d["gpayloads"]), case
        assert np.array_equal(idx.bitmap, d["bitmap"]), case
        slots0 = oracle.grmi_predict_slots(idx, d["probes"])
        assert np.array_equal(slots0, d["slots0"]), case
        slot, probes = oracle.exp_search(idx.gkeys, slots0, d["probes"])
        assert np.array_equal(slot, d["out_slot"]), case
        assert np.array_equal(probes, d["out_probes"]), case
        left, count = oracle.match_runs(idx, slot, d["probes"])
        assert np.array_equal(count > 0, d["found"]), case
        assert int(count.sum()) == d["pairs_r"].size, case
        cnt, s, x, steps = oracle.grmi_join(idx, d["probes"], d["probe_payloads"], threads=1)
        assert (cnt, s, x) == tuple(int(v) for v in d["checksum"]), case
        assert steps == int(d["stats"][0]), case


def test_grmi_layout_appendix_a_example():
    """[5,5,5,9,20] at g=2."""
    keys = np.array([5, 5, 5, 9, 20], np.uint64)
    idx = oracle.grmi_build(keys, np.arange(1, 6, dtype=np.uint64), 2.0, 2,
                            model=oracle.rmi_fit(keys, 2))
    assert idx.gkeys.tolist() == [5, 5, 5, 5, 5, 5, 9, 9, 20, 20]
    assert idx.bitmap.astype(int).tolist() == [1, 1, 1, 0, 0, 0, 1, 0, 1, 0]


def test_spline_hash_build_and_join(golden):
    """learned_hash.py:35-96: identical chains (insertion order) and join."""
    g = golden("spline_hash")
    for case, d in g.items():
        n = d["keys"].size
        sp = spline_from_fixture(d, n, int(d["max_error"]), int(d["radix_bits"]))
        fit = oracle.spline_fit(np.sort(d["keys"]), int(d["max_error"]), int(d["radix_bits"]))
        assert np.array_equal(fit.spline_keys, sp.spline_keys), case
        idx = oracle.spline_hash_build(d["keys"], d["payloads"], table_factor=float(d["table_factor"]),
                                       model=sp)
        assert idx.table_len == int(d["table_len"]), case
        assert np.array_equal(idx.keys, d["e_keys"]), case
        assert np.array_equal(idx.payloads, d["e_payloads"]), case
        if "starts" in d:
            assert np.array_equal(idx.starts, d["starts"]), case
        got = oracle.spline_hash_join(idx, d["probes"], d["probe_payloads"], threads=1)
        assert got == tuple(int(v) for v in d["checksum"]), case
        counts = np.diff(idx.starts)
        frac = (n - np.count_nonzero(counts)) / n
        assert frac == pytest.approx(float(d["collision_fraction"]), abs=0)


def test_lsj_join_matches_reference(golden):
    """lsj.py:95-405: given the reference's sample models, identical
    checksums and sort counters; with the oracle's own fit, identical
    checksums (model neutrality)."""
    g = golden("lsj")
    for case, d in g.items():
        mr = rmi_from_fixture(d, "mr_")
        ms = rmi_from_fixture(d, "ms_")
        w, f = int(d["workers"]), int(d["fanout"])
        res, stats = oracle.lsj_join(d["r_keys"], d["r_payloads"], d["s_keys"], d["s_payloads"],
                                     workers=w, fanout=f, models=(mr, ms))
        assert res == tuple(int(v) for v in d["checksum"]), case
        assert stats == tuple(int(v) for v in d["sort_stats"]), case
        res2, _ = oracle.lsj_join(d["r_keys"], d["r_payloads"], d["s_keys"], d["s_payloads"],
                                  workers=w, fanout=f, sample_rate=float(d["sample_rate"]),
                                  seed=int(d["seed"]))
        assert res2 == res, case


def test_ground_truth_joins_agree(golden):
    g = golden("algos")
    for case, d in g.items():
        want = tuple(int(v) for v in d["checksum"])
        args = (d["r_keys"], d["r_payloads"], d["s_keys"], d["s_payloads"])
        assert oracle.smj_checksum(*args) == want, case
        assert oracle.nlj_checksum(*args) == want, case


def test_rmi_inlj_matches_reference(golden):
    """baselines.py:96-157 (rmi-inlj): the oracle over the
    reference's sorted R and its own fitted model gives the reference's
    checksum and search_steps (the counter is chunking-independent)."""
    for case, d in golden("algos").items():
        m = rmi_from_fixture(d, "rmi_")
        order = np.argsort(d["r_keys"], kind="stable")
        rk, rp = d["r_keys"][order], d["r_payloads"][order]
        got = oracle.rmi_inlj(m, rk, rp, d["s_keys"], d["s_payloads"])
        assert got[:3] == tuple(int(v) for v in d["checksum"]), case
        for w in (1, 4):
            assert got[3] == int(d[f"rmi-inlj_w{w}_counters"][0]), (case, w)
