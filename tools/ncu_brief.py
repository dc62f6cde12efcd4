"""Compact comparison of ncu reports: time, instructions, issue, pipes, L1/L2/DRAM, stall reasons.

  python tools/ncu_brief.py REPORT.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("time_us", "gpu__time_duration.sum", None),
    ("inst_M", "smsp__inst_executed.sum", 1e-6),
    ("issue%", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("warps%", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("fp64%", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("xu%", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1),
    ("alu%", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", 1),
    ("lsu%", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", 1),
    ("l1wave%", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", 1),
    ("l1_smem_wave_M", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1e-6),
    ("l1_hit%", "l1tex__t_sector_hit_rate.pct", 1),
    ("l2_hit%", "lts__t_sector_hit_rate.pct", 1),
    ("l2%", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("dram%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("dram_rd_GB", "dram__bytes_read.sum", 1),
    ("dram_wr_GB", "dram__bytes_write.sum", 1),
    ("ld_req_M", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", 1e-6),
    ("ld_sect_M", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", 1e-6),
]


UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
        "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}


def load(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    d = dict(zip(rows[0], rows[2]))
    for k, u in zip(rows[0], rows[1]):
        if u in UNIT:  # normalise times to us and bytes to GB
            try:
                d[k] = str(float(d[k].replace(",", "")) * UNIT[u])
            except ValueError:
                pass
    return d


def num(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return float("nan")


reps = sys.argv[1:]
data = [load(r) for r in reps]
print(f"{'':22s}" + "".join(f"{r.split('/')[-1][:22]:>24s}" for r in reps))
for name, key, sc in KEYS:
    print(f"{name:22s}" + "".join(f"{num(d.get(key, 'nan')) * (sc or 1):24.3f}" for d in data))
stall = sorted({k for d in data for k in d if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio")})
for k in stall:
    vals = [num(d.get(k, "nan")) for d in data]
    if max(vals) < 0.05:
        continue
    print(f"{k.replace('smsp__average_warp_latency_issue_stalled_', 'st_')[:22]:22s}" + "".join(f"{v:24.3f}" for v in vals))
