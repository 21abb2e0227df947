"""Leaf-product kernel probe (diagnostics): the c5 workload (or a smaller n
of the same decay) in f32 (default) or f64, K3 time and TFLOP/s per multiply.

    python tools/k3_probe.py [n] [reps] [f32|f64]   (env SPAMM_* switches as usual)"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
f64 = len(sys.argv) > 3 and sys.argv[3] == "f64"
cfg = workloads.DEVICE_CONFIGS["c5"]
at = workloads.exponential_decay_device(n, cfg["lam"], cfg["seed"], "cuda",
                                       torch.float64 if f64 else torch.float32)
a = sp.from_device_pointer(at.data_ptr(), n, leaf_size=cfg["leaf"],
                           dtype=np.float64 if f64 else np.float32)
del at
torch.cuda.empty_cache()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(reps):
    for tau in cfg["taus"]:
        flush.zero_()
        torch.cuda.synchronize()
        c, st, det = sp.spamm_detailed(a, a, sp.SpammConfig(tau=tau))
        del c
        fl = 2 * cfg["leaf"] ** 3 * st.leaf_matmuls
        print(f"n={n} tau={tau} retained={st.leaf_matmuls} total={det.ms_total:.3f} ms "
              f"gemm={det.ms_gemm:.3f} ms K3={fl / det.ms_gemm / 1e9:.1f} TFLOP/s", flush=True)
