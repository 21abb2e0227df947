"""Tree construction (from_dense on device data: D2D copy + K1 + pyramid) for one
config; used under ncu for the norm kernel's HBM evidence.  usage: build_probe.py c2|c5"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
if name in workloads.DEVICE_CONFIGS:
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
    print(f"{name}: n={n} from_device (copy + norms + pyramid) {ms:.3f} ms, "
          f"{n * n * 8 * 3 / (ms * 1e-3) / 1e9:.0f} GB/s of copy+read traffic", flush=True)
    del t
