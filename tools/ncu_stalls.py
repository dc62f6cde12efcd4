"""Warp stall reasons (warps per issue-active cycle) of ncu reports, side by side.
  python tools/ncu_stalls.py A.ncu-rep [B.ncu-rep ...]"""
import csv
import io
import subprocess
import sys

cols = {}
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    d = {}
    for h, v in zip(r[0], r[2]):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                d[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
            except ValueError:
                pass
    cols[rep.split("/")[-1]] = d
keys = sorted({k for d in cols.values() for k, v in d.items() if v > 0.05})
print(f"{'':24s}" + "".join(f"{c[:24]:>26s}" for c in cols))
for k in keys:
    print(f"{k:24s}" + "".join(f"{cols[c].get(k, 0.0):26.3f}" for c in cols))
