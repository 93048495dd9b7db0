"""Stall samples and executed instructions per CUDA source line of one kernel
(ncu --page source, SASS correlated with -lineinfo).
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "-c", "1", "--page", "source", "--csv",
                      "--print-source", "sass,cuda"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, ins, src = collections.Counter(), collections.Counter(), {}
h, cur, fname = None, None, ""
for r in rows:
    if r and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        h = r
        iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        continue
    if h is None or len(r) < len(h):
        continue
    if not r[0].isdigit():
        continue  # SASS rows repeat their CUDA line's totals
    cur = (fname, int(r[0]))
    src[cur] = r[1]
    try:
        agg[cur] += int(r[iS].replace(",", "") or 0)
        ins[cur] += int(r[iE].replace(",", "") or 0)
    except ValueError:
        pass
tot = sum(agg.values()) or 1
for key, c in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    f, ln = key
    print(f"{f}:{ln:<5d} {100 * c / tot:5.1f}% ins={ins[key]:>11d}  {src.get(key, '').strip()[:80]}")
