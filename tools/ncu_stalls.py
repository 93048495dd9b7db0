"""Stall samples by reason and opcode for one kernel of an ncu report.
usage: python tools/ncu_stalls.py report.ncu-rep kernel_regex"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "-c", "1", "--page", "source", "--csv",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]


def num(x):
    try:
        return int(x.replace(",", ""))
    except ValueError:
        return 0


isrc = h.index("Source")
reasons = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
tot = {n: collections.Counter() for n in reasons}
for r in data:
    if len(r) < len(h):
        continue
    parts = r[isrc].split()
    if not parts:
        continue
    op = (parts[1] if parts[0].startswith("@") else parts[0]).split(".")[0]
    for n in reasons:
        tot[n][op] += num(r[h.index(n)])
allv = sum(sum(c.values()) for c in tot.values())
for n, c in sorted(tot.items(), key=lambda kv: -sum(kv[1].values())):
    s = sum(c.values())
    if s:
        print(f"{n:<22} {100.0 * s / allv:5.1f}%  {c.most_common(6)}")
