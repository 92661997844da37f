"""Per-kernel warp-stall breakdown (average warps stalled per issue, by
reason) from an ncu report: python tools/stalls.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
pre = "smsp__average_warps_issue_stalled_"
for r in rows[2:]:
    d = dict(zip(h, r))
    st = sorted(((float(v.replace(",", "") or 0), k[len(pre):].replace("_per_issue_active.ratio", ""))
                 for k, v in d.items() if k.startswith(pre)), reverse=True)
    print(d["Kernel Name"][:60])
    print("   " + ", ".join(f"{k} {v:.2f}" for v, k in st[:8] if v > 0.05))
