"""Summarise an LJ_STAGE_TRACE file of the staged GRMI probe."""
import sys

import numpy as np

t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 8).astype(np.float64)
t = t[t[:, 1] > 0]
dur = t[:, 1] - t[:, 0]
print(f"pieces {len(t)}  mean piece {dur.mean() / 1e3:.1f} us  staging share {t[:, 6].sum() / dur.sum():.3f}  "
      f"windows staged/piece {t[:, 3].mean():.2f}  small-window pieces {t[:, 4].mean():.3f}")
span = (t[:, 1].max() - t[:, 0].min()) / 1e6
per_sm = {}
for row in t:
    per_sm[int(row[2])] = per_sm.get(int(row[2]), 0) + row[1] - row[0]
busy = np.array(list(per_sm.values())) / 1e6
print(f"kernel span {span:.3f} ms  per-SM busy min {busy.min():.3f} mean {busy.mean():.3f} max {busy.max():.3f} ms")
