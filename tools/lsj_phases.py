"""Phase breakdown of one LSJ run on a BASELINE config (diagnostics)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2111_08824_b200 as lj  # noqa: E402
from paper_2111_08824_b200 import configs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 0
inp = configs.CONFIGS[cfg](scale=scale)
c = lj.LsjConfig(workers=1, fanout=inp.opts["fanout"], sample_rate=inp.opts["sample_rate"])
for i in range(3):
    torch.cuda.synchronize()
    res, br = lj.lsj_join(inp.r, inp.s, c)
    print(json.dumps({"run": i, "checksum": res.checksum, **br.as_dict(), **br.extra}))
