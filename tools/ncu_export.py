"""Export an .ncu-rep (--set full) into the committed summaries:
profiles/<tag>_details.csv (ncu details page) and traffic_<cfg>.json (per
launch: time, DRAM bytes, issue activity, ...; dram_bytes_per_launch of the
dominant kernel).

    python tools/ncu_export.py rep cfg tag dominant_regex [outdir]
"""
import csv
import io
import json
import re
import subprocess
import sys

rep, cfg, tag, dom = sys.argv[1:5]
outdir = sys.argv[5] if len(sys.argv) > 5 else "profiles"
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
launches = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    e = {"kernel": d.get("Kernel Name", "")}
    for m in M:
        if m in d:
            e[m] = d[m]
            e[m + "_unit"] = u.get(m, "")
    launches.append(e)


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)
    return float(str(v).replace(",", "")) * scale


dl = [e for e in launches if re.search(dom, e["kernel"])]
per = None
if dl:
    tot = [to_bytes(e["dram__bytes_read.sum"], e["dram__bytes_read.sum_unit"]) +
           to_bytes(e["dram__bytes_write.sum"], e["dram__bytes_write.sum_unit"]) for e in dl]
    per = sum(tot) / len(tot)
json.dump({"config": cfg, "source": f"ncu --set full --clock-control none capture ({tag}); dominant = /{dom}/",
           "launches": launches, "dram_bytes_per_launch": per}, open(f"{outdir}/traffic_{cfg}.json", "w"), indent=1)
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
open(f"{outdir}/{tag}_details.csv", "w").write(det)
print(cfg, len(launches), "launches; dominant dram bytes/launch", per)
