"""Summarise an ncu report (raw page) into the numbers we track: time, DRAM bytes, issue, fp64
pipe, occupancy, and an executed-opcode histogram from the source page."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
WANT = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]
for r in rows[2:]:
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            print(f"{w:70s} {r[i]} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
h = srows[1]
ia, isrc = h.index("Instructions Executed"), h.index("Source")
c = Counter()
tot = 0
for r in srows[2:]:
    if len(r) <= ia or not r[ia].isdigit():
        continue
    toks = r[isrc].split()
    op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
    c[op.split(".")[0]] += int(r[ia])
    tot += int(r[ia])
print("executed warp instructions", tot)
print(" ".join(f"{op}:{n / tot * 100:.1f}%" for op, n in c.most_common(22)))
