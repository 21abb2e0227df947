"""Per-multiply device timings for one BASELINE config (diagnostics; set the
SPAMM_*_TIMELINE env vars for per-CTA detail).  usage: probe_cfg.py c3_l2 [traversal]"""
import sys
sys.path.insert(0, ".")
import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
trav = sys.argv[2] if len(sys.argv) > 2 else "auto"
a_h, b_h, leaf, taus = workloads.make_config(name)
a = sp.from_dense(a_h, leaf_size=leaf)
b = a if b_h is a_h else sp.from_dense(b_h, leaf_size=leaf)
import torch
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(2):
    for tau in taus:
        flush.fill_(rep)  # L2 flushed before every multiply, as bench.py does
        torch.cuda.synchronize()
        c, st, det = sp.spamm_detailed(a, b, sp.SpammConfig(tau=tau), traversal=trav)
        if rep == 1:
            print(name, trav, tau, "cull %.3f gemm %.3f ctree %.3f total %.3f" % (
                det.ms_cull, det.ms_gemm, det.ms_ctree, det.ms_total),
                [round(x, 1) for x in det.traverse_phase_us], det.tier_candidates, flush=True)
