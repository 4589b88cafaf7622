"""One step of the bench hot path for a config (for ncu captures).

    python tools/one_step.py c2 [variant] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
variant = sys.argv[2] if len(sys.argv) > 2 else bench.DEFAULT_VARIANT.get(cfg, "direct")
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
torch.cuda.set_device(0)
inp = bench.make_inputs(cfg)
index = bench.build_index(inp)
st = bench.make_step(inp, index, variant)
out = torch.zeros(4, dtype=torch.int64, device="cuda")
for _ in range(reps):
    st(out)
torch.cuda.synchronize()
print(cfg, variant, out.tolist())
