import numpy as np, torch
import paper_2111_08824_b200 as lj
from paper_2111_08824_b200 import configs
inp = configs.config3()
idx = lj.SplineHashIndex(32, 18, 4.0).fit(inp.r)
m = idx.model
print("K", m.spline_keys.size, "aux", None if m._d_aux is None else m._d_aux.numel(), "sub", None if m._d_sub is None else m._d_sub.numel())
st = idx.starts.cpu().numpy().astype(np.int64)
ch = np.diff(st)
print("buckets", ch.size, "nonempty", (ch > 0).sum(), "mean chain (nonempty)", ch[ch > 0].mean(), "max", ch.max())
print("chain hist", np.bincount(np.minimum(ch, 10)))
