"""Per-source-line totals from `ncu -i X --page source --csv --print-source=cuda,sass`."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
fn = None
hdr = None
agg = defaultdict(lambda: [0, 0, 0, ""])
stall_cols = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fn = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[0] == "Function Name":
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")] or 0)
        st = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        te = int(r[hdr.index("Thread Instructions Executed")] or 0)
    except ValueError:
        continue
    if r[0] == "":
        continue
    key = (fn, int(r[0]))
    a = agg[key]
    a[0] += ie
    a[1] += st
    a[2] += te
    a[3] = r[1][:90]
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp instr {tot_i:.3e}, samples {tot_s}")
by = sys.argv[2] if len(sys.argv) > 2 else "instr"
idx = 0 if by == "instr" else 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][idx])[:45]:
    print(f"{k[0]:>16}:{k[1]:<5} instr {100 * v[0] / tot_i:5.1f}%  stall {100 * v[1] / tot_s:5.1f}%  "
          f"lanes {v[2] / max(v[0], 1):5.1f}  {v[3]}")
