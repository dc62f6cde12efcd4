"""Summarise a GPU round's ncu outputs into profiles/ (tracked):
  profiles/<tag>_launches.txt   every launch of the bench command with its device time and share
  profiles/<tag>_edge_ncu.txt   key metrics + stall reasons + executed-opcode mix of the edge kernel
  profiles/traffic.json         DRAM bytes per launch of the edge kernel (bench.py's roofline.traffic)
  python tools/summarize_profiles.py <tag> [<launches.csv> <report.ncu-rep>]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import Counter, defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def launches(tag, path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    ik, iv, ig, ib = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size"), h.index("Block Size")
    tot = defaultdict(float)
    cnt = Counter()
    lines = []
    for r in rows[1:]:
        name = r[ik].split("(")[0].replace("void ", "")
        ns = float(r[iv])
        tot[name] += ns
        cnt[name] += 1
        lines.append(f"{r[0]:>4} {ns / 1e3:10.1f} us  grid {r[ig]:>14} block {r[ib]:>14}  {r[ik][:110]}")
    allns = sum(tot.values())
    out = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold, serialised) of "
           f"`python bench.py --steps 3 --warmup 3 --no-cpu`; {len(lines)} launches", "",
           "## share of device time by kernel"]
    for name, ns in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{ns / allns * 100:6.2f}%  {cnt[name]:3d} launches  {ns / cnt[name] / 1e3:10.1f} us/launch  {name}")
    out += ["", "## launches"] + lines
    open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(out) + "\n")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "sm__cycles_elapsed.avg.per_second"]


def edge(tag, rep, key):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    out = [f"# ncu --set full --clock-control none of the edge pass on the bench workload "
           f"(tools/prof_edge.py, C5, k=8, p=1.2): {v[h.index('Kernel Name')]}", ""]
    vals = {}
    for w in WANT:
        if w in h:
            i = h.index(w)
            out.append(f"{w:70s} {v[i]} {u[i]}")
            vals[w] = (v[i], u[i])
    out += ["", "## stall reasons (warps per issue-active cycle)"]
    for i, x in enumerate(h):
        if x.startswith("smsp__average_warps_issue_stalled") and x.endswith("per_issue_active.ratio"):
            try:
                if float(v[i]) > 0.05:
                    out.append(f"{x.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):24s} {v[i]}")
            except ValueError:
                pass
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    sh = srows[1]
    ia, isrc = sh.index("Instructions Executed"), sh.index("Source")
    c = Counter()
    for r in srows[2:]:
        if len(r) > ia and r[ia].isdigit():
            t = r[isrc].split()
            op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
            c[op.split(".")[0]] += int(r[ia])
    tot = sum(c.values())
    out += ["", f"## executed warp instructions by opcode (total {tot})",
            "  ".join(f"{op}:{n / tot * 100:.1f}%" for op, n in c.most_common(25))]
    open(os.path.join(PROF, f"{tag}_edge_ncu.txt"), "w").write("\n".join(out) + "\n")
    # traffic per launch for bench.py
    tp = os.path.join(PROF, "traffic.json")
    t = json.load(open(tp)) if os.path.exists(tp) else {}
    rb = float(vals["dram__bytes_read.sum"][0]) * (1e9 if vals["dram__bytes_read.sum"][1] == "Gbyte" else 1e6)
    wb = float(vals["dram__bytes_write.sum"][0]) * (1e9 if vals["dram__bytes_write.sum"][1] == "Gbyte" else 1e6)
    t[key] = rb + wb
    json.dump(t, open(tp, "w"), indent=1)


if __name__ == "__main__":
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    lc = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    rep = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "gpurun_out", f"prof_edge_{tag}.ncu-rep")
    if os.path.exists(lc):
        launches(tag, lc)
    if os.path.exists(rep):
        edge(tag, rep, "C5-tile-sparse")
    print("wrote profiles for", tag)
