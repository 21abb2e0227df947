"""Per-rank cost of the row-sharded multiply, measured shard by shard on one
GPU (the ranks of the multi-GPU layout are independent: no collective in the
data path), for W = 1, 2, 4, 8 shards: the slowest shard's device time bounds
the W-GPU step.  usage: python tools/shard_scaling.py c5|c2"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import distributed as spd
from paper_1011_3534_b200 import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
if name in workloads.DEVICE_CONFIGS:
    at, _, leaf, taus = workloads.make_config_device(name, "cuda:0")
    n = at.shape[0]
    a = sp.from_device_pointer(at.data_ptr(), n, leaf_size=leaf)
    del at
    torch.cuda.empty_cache()
else:
    ah, _, leaf, taus = workloads.make_config(name)
    n = ah.shape[0]
    a = sp.from_dense(ah, leaf_size=leaf)
out = {"config": name, "n": n, "taus": list(taus), "per_W": {}}
for W in (1, 2, 4, 8):
    worst, flops = 0.0, 0.0
    per = []
    for r in range(W):
        rows = spd.row_shard(r, W, n, leaf)
        best = None
        for rep in range(3):
            ms = 0.0
            f = 0.0
            for tau in taus:
                c, st, det = sp.spamm_detailed(a, a, sp.SpammConfig(tau=tau), rows=rows)
                ms += det.ms_total
                f += 2.0 * leaf ** 3 * st.leaf_matmuls
                del c
            best = ms if best is None else min(best, ms)
        per.append(best)
        flops += f
        worst = max(worst, best)
    out["per_W"][W] = {"max_rank_ms": worst, "rank_ms": per, "tflops": flops / (worst * 1e-3) / 1e12}
t1 = out["per_W"][1]["max_rank_ms"]
for W in (1, 2, 4, 8):
    out["per_W"][W]["speedup_vs_1"] = t1 / out["per_W"][W]["max_rank_ms"]
print(json.dumps(out))
