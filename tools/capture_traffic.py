"""DRAM traffic per decode launch, tied to the sources being timed.

Run on the GPU box (after the same decode_sweep command ran clean):
    python tools/capture_traffic.py [cfg ...]          (default: 4 2 3; "3g4" = cfg3 at G = 4)
It runs tools/decode_sweep.py --profile under ncu (dram bytes + duration of
every decode kernel launch: the split kernel and the combine), takes the
second (timed) rkv_decode_attention of each config, and writes
profiles/decode_traffic.json with the source hash bench.py checks
(bench.source_hash: the decode .cu/.cuh files), so a stale capture is never
reported as `traffic`.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

cfgs = sys.argv[1:] or ["4", "2", "3"]
log = os.path.join(ROOT, "gpurun_out", "traffic_ncu.csv")
os.makedirs(os.path.dirname(log), exist_ok=True)
cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum", "--clock-control",
       "none", "-k", "regex:decode_(mma|gqa|split|generic)_kernel|decode_combine_kernel", "--csv", "--log-file", log,
       sys.executable, os.path.join(ROOT, "tools", "decode_sweep.py"), "--profile", *cfgs]
subprocess.run(cmd, check=True)
text = open(log).read()
text = text[text.index('"ID"'):]  # skip ncu's preamble lines
rows = list(csv.DictReader(io.StringIO(text)))
launches = {}
for r in rows:
    try:
        lid = int(r["ID"])
    except (KeyError, ValueError):
        continue
    d = launches.setdefault(lid, {"kernel": r["Kernel Name"], "bytes": 0.0, "ns": 0.0})
    unit, val = r["Metric Unit"], float(r["Metric Value"].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    if r["Metric Name"].startswith("dram__bytes"):
        d["bytes"] += val * scale.get(unit, 1)
    elif r["Metric Name"] == "gpu__time_duration.sum":
        d["ns"] = val * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(unit, 1)
order = [launches[k] for k in sorted(launches)]
# per config: (warm-up split + combine) then (timed split + combine)
out = {"capture": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum, tools/decode_sweep.py --profile "
                  f"{' '.join(cfgs)} (second launch of each config: split kernel + combine)",
       "source_hash": bench.source_hash(), "workloads": {}}
per = len(order) // len(cfgs)
for i, c in enumerate(cfgs):
    grp = order[i * per:(i + 1) * per]
    timed = grp[per // 2:]
    out["workloads"]["cfg" + c.replace("g", "_g")] = {"dram_bytes_per_launch": sum(x["bytes"] for x in timed),
                                   "kernels": [{"kernel": x["kernel"][:80], "dram_bytes": x["bytes"],
                                                "ns_cold": x["ns"]} for x in timed]}
# profiles/ (commit it) and gpurun_out/ (the copy a remote run brings back)
for dst in (os.path.join(ROOT, "profiles", "decode_traffic.json"), os.path.join(ROOT, "gpurun_out", "decode_traffic.json")):
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
