"""A/B timing of the leaf-product kernel on c2 (median of repeated multiplies)."""
import os, sys, statistics
sys.path.insert(0, '.')
import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import workloads
a_h, _, leaf, taus = workloads.make_config("c2")
a = sp.from_dense(a_h, leaf_size=leaf)
import torch
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for tau in taus:
    g, tot, tr, ct = [], [], [], []
    for rep in range(12):
        flush.zero_(); torch.cuda.synchronize()
        c, st, det = sp.spamm_detailed(a, a, sp.SpammConfig(tau=tau))
        if rep >= 2:
            g.append(det.ms_gemm); tot.append(det.ms_total); tr.append(det.ms_cull); ct.append(det.ms_ctree)
    print(f"{os.environ.get('TAG','')} tau={tau:.0e} gemm_med={statistics.median(g)*1e3:.1f}us "
          f"total_med={statistics.median(tot)*1e3:.1f}us traverse={statistics.median(tr)*1e3:.1f} ctree={statistics.median(ct)*1e3:.1f} "
          f"TF_gemm={2*64**3*st.leaf_matmuls/statistics.median(g)/1e9:.1f}")
