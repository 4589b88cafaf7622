"""LSJ sort diagnostics per config: oversized sub-buckets, fallbacks, phase times."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_08824_b200 as lj  # noqa: E402
from paper_2111_08824_b200 import configs  # noqa: E402

torch.cuda.set_device(0)
for name, fn in (("c4", lambda: configs.config4()), ("c5s3", lambda: configs.config5(scale=3))):
    inp = fn()
    cfg = lj.LsjConfig(fanout=4096, sample_rate=0.01)
    for rep in range(3):
        res, br = lj.lsj_join(inp.r, inp.s, cfg, counters=False)
        c = res.checksum
    print(json.dumps({"cfg": name, "extra": br.extra, "smpl": br.smpl, "part": br.part, "sort": br.sort,
                      "join": br.join, "count": c[0]}), flush=True)
    del inp
    torch.cuda.empty_cache()
