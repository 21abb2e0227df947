"""Per-rank cost of bench.py's multi-GPU step (the tau sweep partitioned by
distributed.sweep_plan: each tau whole or split into C block-row shards),
measured piece by piece on one GPU -- the ranks are independent (no collective
in the data path), so the slowest rank's summed device time bounds the W-GPU
step.  usage: python tools/sweep_scaling.py c2 [W ...]"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import distributed as spd
from paper_1011_3534_b200 import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
Ws = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
ah, bh, leaf, taus = workloads.make_config(name)
n = ah.shape[0]
a = sp.from_dense(ah, leaf_size=leaf)
b = a if bh is None or bh is ah else sp.from_dense(bh, leaf_size=leaf)
nb = spd.padded_blocks(n, leaf)
row_counts = []
for tau in taus:
    _, _, det = sp.spamm_detailed(a, b, sp.SpammConfig(tau=tau), keep_triples=True)
    row_counts.append(np.bincount(det.triples[:, 0], minlength=nb)[:nb])
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
cache = {}


def piece_ms(q, rows):
    key = (q, rows)
    if key not in cache:
        best = None
        for rep in range(5):
            flush.zero_()
            torch.cuda.synchronize()
            c, st, det = sp.spamm_detailed(a, b, sp.SpammConfig(tau=taus[q]),
                                           rows=None if rows == (0, nb) else rows)
            del c
            if rep:
                best = det.ms_total if best is None else min(best, det.ms_total)
        cache[key] = (best, 2.0 * leaf ** 3 * st.leaf_matmuls)
    return cache[key]


out = {"config": name, "n": n, "taus": list(taus), "per_W": {}}
for W in Ws:
    plan, _ = spd.sweep_plan(W, n, leaf, row_counts)
    rank_ms, flops = [], 0.0
    for pieces in plan:
        ms = 0.0
        for q, rows in pieces:
            t, f = piece_ms(q, tuple(rows))
            ms += t
            flops += f
        rank_ms.append(ms)
    worst = max(rank_ms)
    out["per_W"][W] = {"max_rank_ms": worst, "rank_ms": rank_ms,
                       "plan": [[(float(taus[q]), list(r)) for q, r in p] for p in plan],
                       "tflops": flops / (worst * 1e-3) / 1e12}
t1 = out["per_W"][Ws[0]]["max_rank_ms"]
for W in Ws:
    out["per_W"][W]["speedup_vs_first"] = t1 / out["per_W"][W]["max_rank_ms"]
print(json.dumps(out))
