"""Print the decode plan (kernel, splits, CTAs per SM, ...) for the BASELINE
decode configs and their rank shards: python tools/plan_info.py"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_16383_b200 as P  # noqa: E402
from paper_2501_16383_b200 import sharding  # noqa: E402
from paper_2501_16383_b200 import workload as WL  # noqa: E402

for kv in filter(None, os.environ.get("RKV_OPT", "").split(",")):  # experiment switches
    k_, v_ = kv.split("=")
    P.set_debug_option(k_, int(v_))
for cfg_id, g in ((1, None), (2, None), (3, None), (3, 4), (4, None)):
    w = WL.CONFIGS[cfg_id]
    if g:
        w = dataclasses.replace(w, heads_per_group=g)
    for world in (1, 2, 4, 8):
        _, b = sharding.batch_shard(w.batch, world, 0)
        if b < 1:
            continue
        cfg = P.LayerConfig(batch=b, num_q_heads=w.num_q_heads, num_kv_heads=w.num_kv_heads,
                            heads_per_group=w.heads_per_group, max_tokens=w.tokens, rope_base=w.rope_base)
        print(json.dumps({"cfg": cfg_id, "g": w.heads_per_group, "world": world, "B": b,
                          **P.decode_plan_info(cfg, w.tokens)}), flush=True)
