"""Size histogram of the LSJ split's sub-buckets for a config (which ones exceed the sort's capacity)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_08824_b200 as lj  # noqa: E402
from paper_2111_08824_b200 import configs  # noqa: E402

torch.cuda.set_device(0)
inp = configs.config4()
cfg = lj.LsjConfig(fanout=4096, sample_rate=0.01)
res, br = lj.lsj_join(inp.r, inp.s, cfg, counters=True)
print({k: v for k, v in br.extra.items()})
