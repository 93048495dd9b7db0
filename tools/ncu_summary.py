"""Summarise an ncu report: key details, stall reasons, per-opcode counts and
top source lines.  usage: python tools/ncu_summary.py report.ncu-rep [units]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
keep = ["Duration", "DRAM Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Achieved Active Warps Per SM", "Theoretical Occupancy", "Executed Instructions", "L1/TEX Cache Throughput",
        "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]
for row in det[1:]:
    if len(row) > 4 and row[-4] in keep:
        print(f"{row[-4]:<40} {row[-2]} {row[-3]}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h, v = raw[0], raw[2]
stalls = []
for i, n in enumerate(h):
    if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued") and v[i] not in ("", "0"):
        stalls.append((int(v[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
    if n in ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
             "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
             "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
             "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
             "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"):
        print(f"{n:<60} {v[i]}")
tot = sum(s for s, _ in stalls)
print("stalls:", ", ".join(f"{n} {s / tot * 100:.0f}%" for s, n in sorted(stalls, reverse=True)[:9]))
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "cuda,sass"))))
start = [i for i, r in enumerate(src) if r and r[0] == "Line No"][0]
hdr = src[start]
ie = hdr.index("Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
cur = None
per_line = defaultdict(int)
per_stall = defaultdict(int)
ops = defaultdict(int)
text = {}
for r in src[start + 1:]:
    if len(r) <= ie:
        continue
    if r[0] != "":
        cur = r[0]
        text[cur] = r[1][:90]
        continue
    try:
        n = int(r[ie])
    except ValueError:
        continue
    per_line[cur] += n
    try:
        per_stall[cur] += int(r[ws])
    except ValueError:
        pass
    t = r[3].split()
    if t:
        o = t[1] if t[0].startswith("@") else t[0]
        ops[o.split(".")[0]] += n
sass = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
st2 = [i for i, r in enumerate(sass) if r and r[0] == "Address"][0]
h2 = sass[st2]
ie2, src2 = h2.index("Instructions Executed"), h2.index("Source")
ops = defaultdict(int)
for r in sass[st2 + 1:]:
    if len(r) <= ie2 or not r[src2].split():
        continue
    t = r[src2].split()
    o = t[1] if t[0].startswith("@") else t[0]
    try:
        ops[o.split(".")[0]] += int(r[ie2])
    except ValueError:
        pass
T = sum(ops.values())
print(f"total warp instructions {T}  ({T / units:.1f} per unit)")
print("opcodes:", ", ".join(f"{k} {v / units:.1f}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:24]))
print("top lines (instr per unit, stall samples; inlined lines may repeat across files):")
for k, n in sorted(per_line.items(), key=lambda x: -x[1])[:30]:
    print(f"  {n / units:8.1f} {per_stall[k]:6d}  {k:>5} {text.get(k, '')}")
