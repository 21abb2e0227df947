import sys; sys.path.insert(0,'.')
import numpy as np, paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import workloads
a_h, _, leaf, taus = workloads.make_config("c2")
a = sp.from_dense(a_h, leaf_size=leaf)
for rep in range(3):
    for tau in taus:
        c, st, det = sp.spamm_detailed(a, a, sp.SpammConfig(tau=tau))
        if rep == 2:
            print(tau, "cull_ms %.3f" % det.ms_cull, "gemm %.3f" % det.ms_gemm, "ctree %.3f" % det.ms_ctree, "total %.3f" % det.ms_total, [round(x,1) for x in det.traverse_phase_us], det.tier_candidates)
