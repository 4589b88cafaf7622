"""C3 grouping experiment: bucket + grouped-probe times for the window
count / bin function selected by the environment (LJ_HASH_BINS,
LJ_HASH_KEYBIN), one JSON line.

    LJ_HASH_BINS=512 LJ_HASH_KEYBIN=1 python tools/exp_c3_bins.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402


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
    import paper_2111_08824_b200 as lj
    from paper_2111_08824_b200 import configs

    torch.cuda.set_device(0)
    scale = int(os.environ.get("EXP_SCALE", "1"))
    t0 = time.time()
    inp = configs.config3(scale=scale)
    idx = lj.SplineHashIndex(32, 18, 4.0).fit(inp.r)
    torch.cuda.synchronize()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    out = torch.zeros(4, dtype=torch.int64, device="cuda")
    keys, pays = inp.s.keys, inp.s.payloads
    n_s = len(inp.s)
    scratch = idx.bucket_scratch(n_s)
    res = {"env": {k: v for k, v in os.environ.items() if k.startswith("LJ_")}, "prep_s": time.time() - t0,
           "nbins": scratch["nbins"]}
    res["bucket_ms"] = timeit(lambda: idx.bucket_records(keys, pays, scratch), flush)
    res["probe_ms"] = timeit(lambda: idx.probe_records(n_s, scratch, out), flush)
    out.zero_()
    idx.bucket_records(keys, pays, scratch)
    idx.probe_records(n_s, scratch, out)
    res["words"] = [int(v) & ((1 << 64) - 1) for v in out.tolist()]
    res["ok"] = res["words"][0] == n_s
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
