"""K3 per-CTA timeline on c2 (SPAMM_GEMM_TIMELINE): start/end spread and busy time."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import workloads

a_h, b_h, leaf, taus = workloads.make_config("c2")
a = sp.from_dense(a_h, leaf_size=leaf)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for it in range(3):
    for tau in taus:
        flush.zero_()
        torch.cuda.synchronize()
        c, st, det = sp.spamm_detailed(a, a, sp.SpammConfig(tau=tau))
        if it == 2:
            print(f"tau={tau:g} retained={st.leaf_matmuls} groups={det.n_groups} gemm={det.ms_gemm*1e3:.1f}us "
                  f"ctree={det.ms_ctree*1e3:.1f}us cull={det.ms_cull*1e3:.1f}us total={det.ms_total*1e3:.1f}us",
                  file=sys.stderr, flush=True)
            ph = det.traverse_phase_us
            print("   traverse phases (us from class. end; [0]=launch->class.): " +
                  " ".join(f"{i}:{v:.1f}" for i, v in enumerate(ph) if v), file=sys.stderr, flush=True)
        del c
