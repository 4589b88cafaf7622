"""Per-kernel device times of one bench step (CUPTI through torch.profiler; no ncu).

    python tools/kprof.py c4 [variant] [steps]
"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
variant = sys.argv[2] if len(sys.argv) > 2 else bench.DEFAULT_VARIANT.get(cfg, "direct")
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
torch.cuda.set_device(0)
inp = bench.make_inputs(cfg)
index = bench.build_index(inp)
st = bench.make_step(inp, index, variant)
out = torch.zeros(4, dtype=torch.int64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for _ in range(2):
    st(out)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        flush.zero_()
        st(out)
    torch.cuda.synchronize()
agg = defaultdict(lambda: [0.0, 0])
for ev in prof.events():
    if ev.device_type == torch.autograd.DeviceType.CUDA:
        a = agg[ev.name[:110]]
        a[0] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
        a[1] += 1
tot = sum(v[0] for v in agg.values())
print(f"{cfg} {variant}: {tot / steps / 1000:.3f} ms of kernels per step")
for name, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:28]:
    print(f"{t / steps / 1000:9.3f} ms  x{c / steps:5.1f}  {name}")
print("words", [int(v) & ((1 << 64) - 1) for v in out.cpu().tolist()])
