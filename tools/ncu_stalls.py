"""Warp stall reasons (per issue-active) of every kernel in an ncu report.
Usage: python tools/ncu_stalls.py rep.ncu-rep [top]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
for r in rows[2:]:
    print("==", r[h.index("Kernel Name")][:90])
    items = [(h[i].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), r[i])
             for i in range(len(h)) if "smsp__average_warps_issue_stalled" in h[i] and h[i].endswith("per_issue_active.ratio")]
    items = sorted(items, key=lambda x: -float(x[1] or 0))
    for k, v in items[:top]:
        print(f"   {float(v):7.3f}  {k}")
