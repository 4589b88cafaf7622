"""CPU analysis of the C3 index geometry (design aid, not product):
spline knots per staging cell of the grouped probe's windows, and the
displacement of every build key from its home slot pair in the probe table.
Uses the host generator + oracle only (no GPU)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle
from oracle import gen

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 1
t0 = time.time()
h = gen.config3(scale=scale)
rk = oracle.sort_u64(h.rk)
n = rk.size
print("gen+sort", n, round(time.time() - t0, 1), "s", flush=True)
m = oracle.spline_fit(rk, 32, 18)
K = m.spline_keys.size
print("knots", K, "keys/knot", n / K, round(time.time() - t0, 1), "s", flush=True)
pos, _, _ = oracle.spline_predict(m, rk)
print("predict", round(time.time() - t0, 1), "s", flush=True)

# probe table displacement: slot_j = j + max_{i<=j}(2 pos_i - i)
t = 2 * pos - np.arange(n, dtype=np.int64)
M = np.maximum.accumulate(t)
disp = (np.arange(n, dtype=np.int64) + M) - 2 * pos
for d in (0, 1, 2, 3, 4, 6, 8, 16, 32, 64):
    print(f"disp >= {d}: {float((disp >= d).mean()):.5f}")
print("disp max", int(disp.max()), "mean", float(disp.mean()))
# by pair rounds: pair index = disp // 2 (probe reads pairs at s0, s0+2, ...)
pr = disp // 2
for d in range(0, 6):
    print(f"pair round {d}: {float((pr == d).mean()):.5f}")

sk = m.spline_keys
for nbw in (512, 1024, 2048):
    for nc in (1024, 2048, 4096):
        hist = np.zeros(64, np.float64)
        worst = 0
        npts_max = 0
        for w in range(nbw):
            a = (w * n) // nbw
            b = ((w + 1) * n) // nbw
            klo = int(rk[a]) if w else int(rk[0])
            khi = int(rk[b] - 1) if w + 1 < nbw else int(rk[n - 1])
            if khi < klo:
                continue
            sh = 0
            while ((khi - klo) >> sh) >= nc:
                sh += 1
            keys_w = rk[a:b]
            # cells of the window's keys, knots per cell
            lbl = int(np.searchsorted(sk, np.uint64(klo), "left"))
            lbh = int(np.searchsorted(sk, np.uint64(khi), "left"))
            npts_max = max(npts_max, lbh - lbl + 2)
            kn = sk[lbl : lbh + 1]
            kc = ((kn - np.uint64(klo)) >> np.uint64(sh)).astype(np.int64)
            kc = kc[(kc >= 0) & (kc <= nc)]
            cnt = np.bincount(kc, minlength=nc + 1)
            c = ((keys_w - np.uint64(klo)) >> np.uint64(sh)).astype(np.int64)
            per_key = cnt[np.clip(c, 0, nc)]
            hh = np.bincount(np.minimum(per_key, 63), minlength=64)
            hist += hh
            worst = max(worst, int(per_key.max()))
        hist /= hist.sum()
        cum = np.cumsum(hist)
        print(f"windows {nbw} cells {nc}: npts_max {npts_max} worst knots/cell {worst}; "
              f"P(knots<=1) {cum[1]:.4f} <=2 {cum[2]:.4f} <=3 {cum[3]:.4f} <=4 {cum[4]:.4f} <=6 {cum[6]:.4f}",
              flush=True)
print("done", round(time.time() - t0, 1), "s")
