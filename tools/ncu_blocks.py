"""Hot straight-line SASS blocks of an ncu report (executed instructions,
opcode mix, stall samples).  usage: python tools/ncu_blocks.py report.ncu-rep [n]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
nshow = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
ia, isrc, iss = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


tot = sum(num(r[ia]) for r in data)
groups = []
for idx, r in enumerate(data):
    n, st, s = num(r[ia]), num(r[iss]), r[isrc].strip()
    if groups and groups[-1][1] == n:
        groups[-1][2].append(s)
        groups[-1][3] += st
    else:
        groups.append([idx, n, [s], st])
print("total executed warp instructions", tot)
for g in sorted(groups, key=lambda g: -g[1] * len(g[2]))[:nshow]:
    ops = collections.Counter()
    for s in g[2]:
        op = s.split()[1] if s.startswith("@") else s.split()[0]
        ops["IMAD.MOV" if op.startswith("IMAD.MOV") else op.split(".")[0]] += 1
    print(f"@{g[0]:5d} exec {g[1]:8d} x {len(g[2]):4d} = {g[1] * len(g[2]) / tot * 100:5.1f}%  stalls {g[3]:6d}  "
          + " ".join(f"{k}:{v}" for k, v in ops.most_common(16)))
