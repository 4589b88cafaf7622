"""C3 experiment: direct vs grouped spline-hash probe, and the L2 fetch
granularity limit (random 16-B reads of chain offsets / entries).

    python tools/exp_c3.py [--scale-s N]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch


def set_l2_fetch(bytes_):
    from cuda.bindings import driver as drv

    torch.cuda.synchronize()
    (err,) = drv.cuCtxSetLimit(drv.CUlimit.CU_LIMIT_MAX_L2_FETCH_GRANULARITY, bytes_)
    err2, v = drv.cuCtxGetLimit(drv.CUlimit.CU_LIMIT_MAX_L2_FETCH_GRANULARITY)
    return int(err), int(v)


def timeit(fn, flush, reps=5):
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    args = ap.parse_args()
    import paper_2111_08824_b200 as lj
    from paper_2111_08824_b200 import configs

    torch.cuda.set_device(0)
    t0 = time.time()
    inp = configs.CONFIGS[args.config]()
    t1 = time.time()
    o = dict(lj.DEFAULT_OPTS, **inp.opts)
    if inp.algorithm == "spline-hash-inlj":
        idx = lj.SplineHashIndex(o["spline_error"], o["radix_bits"], o["table_factor"]).fit(inp.r)
    else:
        idx = lj.GappedRmiIndex(o["gap_factor"], o["rmi_fanout"]).fit(inp.r)
    torch.cuda.synchronize()
    t2 = time.time()
    info = {"gen_s": t1 - t0, "build_s": t2 - t1, "n_r": len(inp.r), "n_s": len(inp.s)}
    if hasattr(idx, "model") and hasattr(idx.model, "spline_keys"):
        info["npts"] = int(idx.model.spline_keys.size)
    print(json.dumps(info), flush=True)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    out = torch.zeros(4, dtype=torch.int64, device="cuda")
    keys, pays = inp.s.keys, inp.s.payloads
    n_s = len(inp.s)
    scratch = idx.bucket_scratch(n_s)
    res = {}
    for g in (128,):
        res[f"direct_{g}"] = timeit(lambda: idx.join_checksum(keys, pays, out=out), flush)
        res[f"bucket_{g}"] = timeit(lambda: idx.bucket_records(keys, pays, scratch), flush)
        res[f"grouped_probe_{g}"] = timeit(lambda: idx.probe_records(n_s, scratch, out), flush)
        print(json.dumps(res), flush=True)
    o1 = torch.zeros(4, dtype=torch.int64, device="cuda")
    o2 = torch.zeros(4, dtype=torch.int64, device="cuda")
    idx.join_checksum(keys, pays, out=o1)
    idx.bucket_records(keys, pays, scratch)
    idx.probe_records(n_s, scratch, o2)
    res["direct_words"] = o1.tolist()
    res["grouped_words"] = o2.tolist()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
