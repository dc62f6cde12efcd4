"""Executed-instruction profile of an ncu report's SASS (source page): instructions and stall
samples per address range, to split the inner edge loop from per-row overhead.

  python tools/ncu_hot.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1] if "Address" not in rows[0] else rows[0]
start = 2 if h is rows[1] else 1
ia = h.index("Instructions Executed")
iaddr = h.index("Address")
isrc = h.index("Source")
samp = [i for i, n in enumerate(h) if n.startswith("Warp Stall Sampling (All")]
recs = []
for r in rows[start:]:
    if len(r) <= ia or not r[ia].strip().isdigit():
        continue
    s = int(r[samp[0]]) if samp and r[samp[0]].strip().isdigit() else 0
    recs.append((int(r[iaddr], 16) if r[iaddr].startswith("0x") else int(r[iaddr]), int(r[ia]), s, r[isrc]))
tot = sum(x[1] for x in recs)
tots = sum(x[2] for x in recs) or 1
print(f"total executed {tot}, stall samples {tots}")
# group consecutive instructions with identical execution counts into blocks
blocks = []
for a, n, s, t in recs:
    if blocks and blocks[-1][2] == n:
        blocks[-1][1] = a
        blocks[-1][3] += 1
        blocks[-1][4] += s
    else:
        blocks.append([a, a, n, 1, s, t])
blocks.sort(key=lambda b: -b[2] * b[3])
for b in blocks[:top]:
    print(f"{b[0]:#07x}-{b[1]:#07x} x{b[2]:>10d} len {b[3]:4d}  inst {b[2] * b[3] / tot * 100:5.1f}%  stall {b[4] / tots * 100:5.1f}%  {b[5][:60]}")
