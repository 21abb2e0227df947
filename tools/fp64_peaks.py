"""Measure the FP64 roofline denominators on the B200 box.

Runs tools/fp64_peaks (DMMA / DFMA microbenchmarks) and times cuBLAS DGEMM
8192^3 through torch.matmul, then writes profiles/fp64_peaks.json.  The bench
reads that file for roofline.peak; MEASURED_PEAKS.json carries no FP64 figure.
"""
import json
import os
import subprocess
import sys

import torch

here = os.path.dirname(os.path.abspath(__file__))
root = os.path.dirname(here)
out = json.loads(subprocess.check_output([os.path.join(here, "fp64_peaks")]).decode())
n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 1e30
for _ in range(5):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
out["cublas_dgemm_8192_ms"] = best
out["cublas_dgemm_8192_tflops"] = 2.0 * n ** 3 / best / 1e9
out["gpu_name"] = torch.cuda.get_device_name(0)
print(json.dumps(out))
os.makedirs(os.path.join(root, "gpurun_out"), exist_ok=True)
with open(os.path.join(root, "gpurun_out", "fp64_peaks.json"), "w") as fh:
    json.dump(out, fh, indent=1)
