"""Top SASS instructions by warp-stall samples for one kernel in an .ncu-rep.
    python tools/ncu_src.py rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}", "-c", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
sk = "Warp Stall Sampling (All Samples)"
tot = sum(float(d[sk] or 0) for d in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {id(d): i for i, d in enumerate(data)}
for d in sorted(data, key=lambda d: -float(d[sk] or 0))[:top]:
    v = float(d[sk] or 0)
    st = sorted(((float(d[s] or 0), s[6:]) for s in stalls), reverse=True)[:3]
    print(f"{100 * v / tot:5.1f}% [{idx[id(d)]:5d}] {d['Source'].strip()[:60]:60s} " +
          " ".join(f"{n}={100 * c / max(v, 1):.0f}" for c, n in st if c))
