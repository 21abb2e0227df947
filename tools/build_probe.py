"""Tree construction (from_dense on device data: D2D copy + K1 + pyramid) for one
config; used under ncu for the norm kernel's HBM evidence.  usage: build_probe.py c2|c5"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
if name.startswith("rand"):  # uniform(0.5, 1.5) entries, n = name[4:]: no tiny values anywhere
    at = torch.rand((int(name[4:]), int(name[4:])), dtype=torch.float64, device="cuda") + 0.5
    leaf = 64
elif name in workloads.DEVICE_CONFIGS:
    at, _, leaf, _ = workloads.make_config_device(name, "cuda:0")
else:
    a_h, _, leaf, _ = workloads.make_config(name)
    at = torch.from_numpy(a_h).cuda()
n = at.shape[0]
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    t = sp.from_device_pointer(at.data_ptr(), n, leaf_size=leaf)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    import os
    fused = os.environ.get("SPAMM_NO_FUSED_BUILD") is None
    traffic = n * n * 8 * (2 if fused else 3)  # fused: read the source once, write the tree
    print(f"{name}: n={n} from_device ({'fused read+write+norms' if fused else 'copy, then norms'}"
          f" + pyramid) {ms:.3f} ms, {traffic / (ms * 1e-3) / 1e9:.0f} GB/s of DRAM traffic, "
          f"algorithmic (one read of n^2 f64) {n * n * 8 / 6534.5e9 * 1e3:.2f} ms at 6534.5 GB/s",
          flush=True)
    if rep == 2 and "check" in sys.argv:
        ref = sp.from_device_pointer(at.data_ptr(), n, leaf_size=leaf) if False else None
    del t
