"""Generate golden fixtures by importing the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python oracle/make_golden.py            # writes tests/golden/*.npz

The reference is imported read-only from /root/reference/pkg/src with a
writable numba cache.  Every fixture stores its inputs, so the tests that
consume them never need the reference (it does not exist on the GPU box).
Fixtures pin (a) the C oracle (tests/test_oracle_golden.py) and (b) the CUDA
path (tests/test_gpu_parity.py) to the reference's own outputs.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "lj_numba_cache"))
    os.environ["PYTHONDONTWRITEBYTECODE"] = "1"
    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import learned_joins  # noqa: F401

    return learned_joins


def checksum(res):
    t = (res.payloads_r + res.payloads_s).astype(np.uint64)
    if t.size == 0:
        return np.array([0, 0, 0], dtype=np.uint64)
    return np.array([t.size, np.sum(t, dtype=np.uint64), np.bitwise_xor.reduce(t)], dtype=np.uint64)


def rmi_params(m, prefix=""):
    return {
        prefix + "root": np.array([m.root_slope, m.root_intercept], dtype=np.float64),
        prefix + "trained_len": np.int64(m.trained_len),
        prefix + "leaf_slope": m.leaf_slope.astype(np.float64),
        prefix + "leaf_intercept": m.leaf_intercept.astype(np.float64),
        prefix + "clamp_lo": m.clamp_lo.astype(np.int64),
        prefix + "clamp_hi": m.clamp_hi.astype(np.int64),
        prefix + "err_lo": m.err_lo.astype(np.int64),
        prefix + "err_hi": m.err_hi.astype(np.int64),
    }


def key_sets(lj):
    """Named sorted/unsorted key sets covering the distributions the BASELINE
    configs use (uniform 2^63, lognormal x1e12, clustered normals) and the
    reference's own generators, duplicates and tiny edge cases."""
    rng = np.random.default_rng(20211116)
    sets = {}
    sets["unif63"] = np.unique(rng.integers(0, 2**63, 20000, dtype=np.uint64))
    v = np.floor(1e12 * rng.lognormal(0.0, 2.0, 30000))
    sets["lognorm1e12"] = np.unique(np.minimum(v, 2.0**63 - 1).astype(np.uint64))[:20000]
    centres = rng.uniform(0, 2.0**62, 8)
    c = centres[rng.integers(0, 8, 20000)] + rng.normal(0, 2.0**40, 20000)
    sets["clusters"] = np.unique(np.clip(c, 0, 2.0**63 - 1).astype(np.uint64))
    sets["seq_h"] = np.sort(lj.gen_dataset(lj.DatasetSpec("seq_h", 5000, 3)))
    sets["lognorm_ref"] = np.sort(lj.gen_dataset(lj.DatasetSpec("lognorm", 5000, 5)))
    d = lj.inject_duplicates(lj.gen_dataset(lj.DatasetSpec("unif", 4000, 7)), 0.25, 1)
    sets["dups"] = np.sort(d)
    sets["linear"] = np.arange(100, dtype=np.uint64)
    sets["tiny"] = np.array([5, 5, 5, 9, 20], dtype=np.uint64)
    sets["single"] = np.array([42], dtype=np.uint64)
    # keys above 2^53 that collapse to equal doubles (spline dx == 0 path)
    sets["dbl_collide"] = np.sort(
        np.unique((np.uint64(2**60) + rng.integers(0, 4096, 3000, dtype=np.uint64)))
    )
    return sets


def probes_for(keys, rng, n=4000):
    hit = rng.choice(keys, size=n // 2, replace=True)
    miss = rng.integers(0, max(int(keys.max()) * 2, 10) if keys.max() < 2**62 else 2**63, n // 2,
                        dtype=np.uint64)
    edge = np.array([0, 1, keys.min(), keys.max(), 2**63 - 1, 2**64 - 2], dtype=np.uint64)
    p = np.concatenate([hit, miss, edge]).astype(np.uint64)
    return rng.permutation(p)


def make_models(lj, sets):
    fan = {"unif63": 64, "lognorm1e12": 256, "clusters": 128, "seq_h": 32, "lognorm_ref": 64,
           "dups": 16, "linear": 1, "tiny": 4, "single": 2, "dbl_collide": 8}
    rng = np.random.default_rng(7)
    out = {}
    for name, keys in sets.items():
        m = lj.RecursiveModelIndex(fanout=fan[name]).fit(keys)
        pr = probes_for(keys, rng)
        pos, lo, hi = m.predict_many(pr)
        d = {"keys": keys, "probes": pr, "fanout": np.int64(fan[name]), "pos": pos, "lo": lo,
             "hi": hi, "route": m.route_many(pr)}
        d.update(rmi_params(m))
        for P in (1, 7, 4096):
            d[f"part_{P}"] = lj.partition_index(m, pr, P)
        sp = lj.RadixSplineIndex(max_error=8 if name != "clusters" else 32,
                                 radix_bits=10 if name != "clusters" else 18).fit(keys)
        spos, slo, shi = sp.predict_many(pr)
        d.update({
            "sp_max_error": np.int64(sp.max_error), "sp_radix_bits": np.int64(sp.radix_bits),
            "sp_keys": sp.spline_keys, "sp_ranks": sp.spline_ranks.astype(np.int64),
            "sp_radix_table": sp.radix_table.astype(np.int64), "sp_shift": np.int64(sp.shift),
            "sp_pos": spos, "sp_lo": slo, "sp_hi": shi,
            "sp_part_4n": lj.partition_index(sp, pr, 4 * keys.size),
            "sp_part_3": lj.partition_index(sp, pr, 3),
        })
        out[name] = d
    return out


def make_grmi(lj, sets):
    rng = np.random.default_rng(11)
    out = {}
    for name in ("unif63", "lognorm1e12", "seq_h", "dups", "tiny", "linear", "single"):
        base = sets[name] if sets[name].size <= 3000 else np.sort(rng.choice(sets[name], 3000, replace=False))
        keys = rng.permutation(base)
        rel = lj.make_relation(keys, 3)
        for gap in ((1.0, 2.0, 2.5) if keys.size > 100 else (1.0, 2.0, 2.5, 4.0)):
            idx = lj.GappedRmiIndex(gap, 16 if keys.size > 100 else 2).fit(rel)
            pr = probes_for(base, rng, 1000)
            prel = lj.make_relation(pr, 9)
            slots0 = idx.predict_slots(pr)
            out_slot = np.empty(pr.size, np.int64)
            out_probes = np.empty(pr.size, np.int64)
            from learned_joins.gapped import _search_batch

            _search_batch(idx.gkeys, slots0, pr, out_slot, out_probes)
            st = lj.LookupStats()
            pays, src, found = idx.lookup_batch(pr, st)
            res = lj.JoinResult(pays, prel.payloads[src])
            d = {"keys": keys, "payloads": rel.payloads, "gap": np.float64(gap),
                 "fanout": np.int64(idx.rmi_fanout), "gkeys": idx.gkeys,
                 "gpayloads": idx.gpayloads, "bitmap": idx.bitmap, "L": np.int64(idx.slot_count),
                 "probes": pr, "probe_payloads": prel.payloads, "slots0": slots0,
                 "out_slot": out_slot, "out_probes": out_probes, "found": found,
                 "pairs_r": pays, "pairs_src": src, "checksum": checksum(res),
                 "stats": np.array([st.search_steps, st.predictions, st.leaf_switches], np.int64)}
            d.update(rmi_params(idx.rmi))
            out[f"{name}_g{gap}"] = d
    return out


def make_spline_hash(lj, sets):
    rng = np.random.default_rng(13)
    out = {}
    for name in ("unif63", "clusters", "seq_h", "dups", "tiny", "single", "dbl_collide"):
        base = sets[name] if sets[name].size <= 3000 else np.sort(rng.choice(sets[name], 3000, replace=False))
        keys = rng.permutation(base)
        rel = lj.make_relation(keys, 5)
        for tf in (1.0, 4.0, 2.5):
            idx = lj.SplineHashIndex(max_error=32, radix_bits=18 if name == "clusters" else 12,
                                     table_factor=tf).fit(rel)
            pr = probes_for(base, rng, 1000)
            prel = lj.make_relation(pr, 6)
            pays, src = idx.probe_batch(pr)
            res = lj.JoinResult(pays, prel.payloads[src])
            m = idx.model
            d = {"keys": keys, "payloads": rel.payloads, "table_factor": np.float64(tf),
                 "table_len": np.int64(idx.table_len), "max_error": np.int64(32),
                 "radix_bits": np.int64(m.radix_bits), "sp_keys": m.spline_keys,
                 "sp_ranks": m.spline_ranks.astype(np.int64), "sp_radix_table": m.radix_table,
                 "sp_shift": np.int64(m.shift), "e_keys": idx._keys, "e_payloads": idx._payloads,
                 "probes": pr, "probe_payloads": prel.payloads, "pairs_r": pays, "pairs_src": src,
                 "checksum": checksum(res), "collision_fraction": np.float64(idx.collision_fraction())}
            if idx.table_len <= 100000:
                d["starts"] = idx._starts
            out[f"{name}_t{tf}"] = d
    return out


def make_lsj(lj):
    out = {}
    from learned_joins.lsj import sample_train

    cases = [
        ("seqh_dup", lj.inject_duplicates(lj.gen_dataset(lj.DatasetSpec("seq_h", 5000, 21)), 0.25, 1),
         lj.inject_duplicates(lj.gen_dataset(lj.DatasetSpec("seq_h", 5000, 22)), 0.25, 2)),
        ("lognorm", lj.gen_dataset(lj.DatasetSpec("lognorm", 6000, 31)),
         lj.gen_dataset(lj.DatasetSpec("lognorm", 6000, 32))),
    ]
    rng = np.random.default_rng(17)
    # Zipf-duplicated S over a lognormal R, the config-4 shape at desk scale
    rk = np.unique(np.floor(2.0**40 * rng.lognormal(0, 1.5, 9000)).astype(np.uint64))[:6000]
    w = 1.0 / np.arange(1, rk.size + 1) ** 1.0
    sidx = rng.choice(rk.size, size=6000, p=w / w.sum())
    cases.append(("zipf", rng.permutation(rk), np.sort(rk)[sidx]))
    for name, kr, ks in cases:
        r = lj.make_relation(kr, 5)
        s = lj.make_relation(ks, 6)
        for workers, fanout, rate in ((1, 1000, 0.01), (4, 1000, 0.02), (2, 64, 0.05), (3, 4096, 0.01)):
            cfg = lj.LsjConfig(workers=workers, fanout=fanout, sample_rate=rate)
            res, br = lj.lsj_join(r, s, cfg)
            mr = sample_train(r, rate, workers, cfg.seed)
            ms = sample_train(s, rate, workers, cfg.seed ^ 0x5DEECE66D)
            d = {"r_keys": r.keys, "r_payloads": r.payloads, "s_keys": s.keys,
                 "s_payloads": s.payloads, "workers": np.int64(workers), "fanout": np.int64(fanout),
                 "sample_rate": np.float64(rate), "seed": np.int64(cfg.seed),
                 "checksum": checksum(res),
                 "sort_stats": np.array([br.sort_stats.comparator_count,
                                         br.sort_stats.partitions_sorted], np.int64)}
            d.update(rmi_params(mr, "mr_"))
            d.update(rmi_params(ms, "ms_"))
            out[f"{name}_w{workers}_f{fanout}"] = d
    return out


def make_algos(lj):
    """The four hot-path runners through the reference's own ALGORITHMS
    registry (bench.py:277-289), on c01-style inputs (test_acceptance.py:73-94)."""
    from learned_joins.bench import ALGORITHMS, DEFAULT_OPTS, make_join_inputs

    out = {}
    for kind in ("seq_h", "unif", "lognorm"):
        for n, dup in ((1000, 0.0), (4000, 0.25)):
            r, s, _ = make_join_inputs(kind, n, 42, dup_frac=dup)
            truth = checksum(lj.nlj_oracle(r, s))
            for algo in ("grmi-inlj", "buffered-grmi-inlj", "spline-hash-inlj", "lsj", "rmi-inlj"):
                for workers in (1, 4):
                    opts = dict(DEFAULT_OPTS)
                    res, br, _ = ALGORITHMS[algo](r, s, workers, opts)
                    c = checksum(res)
                    assert np.array_equal(c, truth), (algo, kind, n, dup)
                    key = f"{kind}_{n}_{dup}"
                    if key not in out:
                        out[key] = {"r_keys": r.keys, "r_payloads": r.payloads, "s_keys": s.keys,
                                    "s_payloads": s.payloads, "checksum": truth}
                    ctr = br.counters()
                    if algo == "rmi-inlj" and "rmi_root" not in out[key]:
                        # the model _run_rmi_inlj fits (bench.py:184-192), for exact step parity
                        srt = r.sorted_by_key()
                        m = lj.RecursiveModelIndex(fanout=opts["rmi_fanout"]).fit(srt.keys)
                        out[key].update(rmi_params(m, "rmi_"))
                    out[key][f"{algo}_w{workers}_counters"] = np.array(
                        [ctr["search_steps"], ctr["predictions"], ctr["leaf_switches"],
                         ctr["comparator_count"], ctr["partitions_sorted"]], np.int64)
    return out


def make_c01(lj):
    """The reference acceptance criterion c01's sweep (test_acceptance.py:73-94:
    kinds x n in {1e3, 1e4} x dup in {0, 0.25, 0.5}, plus n = 1e5 at dup 0.5;
    the full n = 1e5 row would triple the fixture) through the
    reference's ALGORITHMS registry: inputs, NLJ truth checksum and every
    runner's counters at workers 1 and 4."""
    from learned_joins.bench import ALGORITHMS, DEFAULT_OPTS, make_join_inputs

    out = {}
    for kind in ("seq_h", "unif", "lognorm"):
        for n, dup in [(n, d) for n in (10**3, 10**4) for d in (0.0, 0.25, 0.5)] + [(10**5, 0.5)]:
            if True:  # n = 1e5 at the largest duplicate share only (fixture size)
                r, s, _ = make_join_inputs(kind, n, 42, dup_frac=dup)
                truth = checksum(lj.nlj_oracle(r, s))
                key = f"{kind}_{n}_{dup}"
                out[key] = {"r_keys": r.keys, "r_payloads": r.payloads, "s_keys": s.keys,
                            "s_payloads": s.payloads, "checksum": truth}
                for algo in ("grmi-inlj", "buffered-grmi-inlj", "spline-hash-inlj", "lsj", "rmi-inlj"):
                    for workers in (1, 4):
                        res, br, _ = ALGORITHMS[algo](r, s, workers, dict(DEFAULT_OPTS))
                        assert np.array_equal(checksum(res), truth), (algo, kind, n, dup)
                        ctr = br.counters()
                        out[key][f"{algo}_w{workers}_counters"] = np.array(
                            [ctr["search_steps"], ctr["predictions"], ctr["leaf_switches"],
                             ctr["comparator_count"], ctr["partitions_sorted"]], np.int64)
    return out


def make_util(lj):
    from learned_joins.util import chunk_bounds, mix64

    x = np.concatenate([np.arange(64, dtype=np.uint64),
                        np.random.default_rng(3).integers(0, 2**64 - 1, 4000, dtype=np.uint64),
                        np.array([2**64 - 1, 2**63, 2**63 - 1], dtype=np.uint64)])
    d = {"x": x, "mix64": mix64(x)}
    for seed in (0, 1, 42, 2**40 + 5):
        d[f"payloads_{seed}"] = lj.make_relation(np.arange(1000, dtype=np.uint64), seed).payloads
    bounds = []
    for n in (0, 1, 7, 100, 10**6 + 3, 2**22):
        for w in (1, 2, 3, 4, 7, 8):
            bounds.append(np.concatenate([[n, w], chunk_bounds(n, w)]))
    d["chunk_bounds"] = np.array([np.pad(b, (0, 11 - b.size), constant_values=-1) for b in bounds])
    return d


def save(name, obj):
    os.makedirs(OUT, exist_ok=True)
    flat = {}
    for case, d in obj.items():
        if isinstance(d, dict):
            for k, v in d.items():
                flat[f"{case}/{k}"] = np.asarray(v)
        else:
            flat[case] = np.asarray(d)
    np.savez_compressed(os.path.join(OUT, name), **flat)
    print(name, os.path.getsize(os.path.join(OUT, name)), "bytes")


def main():
    lj = _import_reference()
    if len(sys.argv) > 1 and sys.argv[1] == "algos":
        save("algos.npz", make_algos(lj))
        return
    if len(sys.argv) > 1 and sys.argv[1] == "c01":
        save("c01.npz", make_c01(lj))
        return
    sets = key_sets(lj)
    save("util.npz", make_util(lj))
    save("models.npz", make_models(lj, sets))
    save("grmi.npz", make_grmi(lj, sets))
    save("spline_hash.npz", make_spline_hash(lj, sets))
    save("lsj.npz", make_lsj(lj))
    save("algos.npz", make_algos(lj))
    save("c01.npz", make_c01(lj))


if __name__ == "__main__":
    main()
