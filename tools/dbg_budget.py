import sys; sys.path.insert(0, '.')
import numpy as np, paper_1011_3534_b200 as sp
from tests.test_gpu_traversal import _decay
n, leaf, tau = 128, 16, 1e-6
a = sp.from_dense(_decay(n, n + leaf), leaf_size=leaf)
b = sp.from_dense(_decay(n, n + leaf + 1, 0.8), leaf_size=leaf)
cfg = sp.SpammConfig(tau=tau, collect_boxes=True)
for rep in range(3):
    r1 = sp.spamm_detailed(a, b, cfg, keep_triples=True)
    r2 = sp.spamm_detailed(a, b, cfg, keep_triples=True, traversal="tiered")
    print(rep, r1[1].omitted_budget, r2[1].omitted_budget, r1[2].tier_pruned, r2[2].tier_pruned,
          [(x.i_lo, x.j_lo, x.k_lo, x.edge, x.tier) for x in r1[1].boxes] == [(x.i_lo, x.j_lo, x.k_lo, x.edge, x.tier) for x in r2[1].boxes])
