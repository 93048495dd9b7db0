"""Per-CTA timeline of the MHA decode kernel (build with
RKV_NVCC_EXTRA=-DRKV_DEC_TRACE): prologue (plan, mask, q RoPE, first TMA
stages) vs tile loop, the spread of CTA end times, by split index and by
SM co-residency."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import decode_sweep  # noqa: E402
import paper_2501_16383_b200 as P  # noqa: E402

for kv in filter(None, os.environ.get("RKV_OPT", "").split(",")):  # experiment switches, e.g. RKV_OPT=decode_splits=40
    k_, v_ = kv.split("=")
    P.set_debug_option(k_, int(v_))
decode_sweep.run(int(sys.argv[1]) if len(sys.argv) > 1 else 2, iters=3)
buf = (ctypes.c_ulonglong * (4096 * 4))()
P.rotatekv.lib().rkv_debug_decode_trace(buf)
t = np.array(buf, dtype=np.int64).reshape(4096, 4)
cid = np.nonzero(t[:, 0])[0]
t = t[cid]
t0 = t[:, 0].min()
end = (t[:, 2] - t0) / 1e3
loop = (t[:, 2] - t[:, 1]) / 1e3
print(f"CTAs {len(t)}: span {end.max():.1f} us; start spread {(t[:, 0].max() - t0) / 1e3:.1f} us")
print(f"prologue median {np.median(t[:, 1] - t[:, 0]) / 1e3:.2f} us; loop pct 0/10/50/90/100: "
      + " ".join(f"{v:.1f}" for v in np.percentile(loop, [0, 10, 50, 90, 100])))
S = int(cid.max() % 1000) if False else None
sms, counts = np.unique(t[:, 3], return_counts=True)
share = dict(zip(sms, counts))
co = np.array([share[s] for s in t[:, 3]])
for c in sorted(set(co)):
    sel = co == c
    print(f"CTAs sharing an SM with {c - 1} other(s): {sel.sum()}, loop median {np.median(loop[sel]):.1f} us, "
          f"max {loop[sel].max():.1f}")
gx = int(os.environ.get("GX", "0"))
if gx:
    split = cid % gx
    for s_ in range(gx):
        sel = split == s_
        print(f"split {s_}: n {sel.sum()} loop median {np.median(loop[sel]):.1f} max {loop[sel].max():.1f}")
# per-SM pairs: (faster, slower) loop time of the two co-resident CTAs
pairs = []
for s_ in sms:
    sel = np.nonzero(t[:, 3] == s_)[0]
    if len(sel) == 2:
        a, b_ = sorted(loop[sel])
        pairs.append((s_, a, b_))
pairs = np.array(pairs)
if len(pairs):
    print("pair fast pct 10/50/90:", " ".join(f"{v:.1f}" for v in np.percentile(pairs[:, 1], [10, 50, 90])),
          "| slow pct 10/50/90:", " ".join(f"{v:.1f}" for v in np.percentile(pairs[:, 2], [10, 50, 90])))
    slow_sms = pairs[pairs[:, 2] > np.percentile(pairs[:, 2], 85)][:, 0].astype(int)
    print("slowest-pair SMs:", sorted(slow_sms.tolist()))
# launch order: the first wave (linear CTA id < number of SMs) vs the rest
nsm = 148
first = cid < nsm
print(f"first-wave CTAs: loop median {np.median(loop[first]):.1f} | later CTAs: {np.median(loop[~first]):.1f}")
# the slowest CTAs: linear id, SM, loop time, and their SM partner's
if os.environ.get("SLOWEST"):
    order = np.argsort(-loop)[: int(os.environ["SLOWEST"])]
    for i in order:
        sm = t[i, 3]
        partner = [j for j in np.nonzero(t[:, 3] == sm)[0] if j != i]
        pl = f"{cid[partner[0]]}:{loop[partner[0]]:.1f}" if partner else "-"
        print(f"cid {cid[i]} sm {sm} loop {loop[i]:.1f} start {(t[i, 0] - t0) / 1e3:.2f} partner {pl}")
