"""BASELINE config 4: SP2/TC2 purification of the 32^3 Morton-ordered cubic
lattice (n = 32768), every square a SpAMM at leaf 64, tau = 1e-7, 30 sweeps,
n_occ = n / 2 -- on one B200, through the drop-in purification driver.
Writes one JSON line (time, retained-leaf TFLOP/s, trace, idempotency error,
energy; with --reference also the tau = 0 run and delta_e_rel).

usage: python tools/c4_purify.py [--L 32] [--sweeps 30] [--tau 1e-7] [--reference]"""
import argparse
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import purification as P
from paper_1011_3534_b200 import workloads

ap = argparse.ArgumentParser()
ap.add_argument("--L", type=int, default=32)
ap.add_argument("--sweeps", type=int, default=30)
ap.add_argument("--tau", type=float, default=1e-7)
ap.add_argument("--leaf", type=int, default=64)
ap.add_argument("--reference", action="store_true")
args = ap.parse_args()

n = args.L ** 3
h = workloads.cubic_lattice_hamiltonian_device(args.L, "cuda:0")
f = sp.from_device_pointer(h.data_ptr(), n, leaf_size=args.leaf)
del h
torch.cuda.empty_cache()


def run(tau, ref=None):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = P.purify(f, n // 2, P.SpammMode(tau), max_iter=args.sweeps,
                   reference_energy=ref if ref is not None else float("nan"))
    torch.cuda.synchronize()
    return res, time.perf_counter() - t0


res, sec = run(args.tau, None)
flops = 2.0 * args.leaf ** 3 * res.total_leaf_matmuls
x = res.density
x2, _ = sp.spamm(x, x, sp.SpammConfig(tau=0.0))
idem = sp.add(x2, sp.scale(x, -1.0)).norm()
line = {
    "workload": f"c4: SP2 on the {args.L}^3 Morton lattice, n={n}, leaf={args.leaf}, "
                f"tau={args.tau}, {args.sweeps} sweeps, n_occ={n // 2}",
    "seconds": sec, "sweeps": args.sweeps,
    "retained_leaf_tflops": flops / sec / 1e12,
    "total_leaf_matmuls": res.total_leaf_matmuls,
    "dense_equivalent_leaf_matmuls_per_sweep": (n // args.leaf) ** 3,
    "step_leaf_matmuls": res.step_leaf_matmuls,
    "final_trace": res.trace_history[-1], "idempotency_error_fro": idem,
    "energy": res.energy,
    "note": "wall time of purify() incl. tree algebra, traces and the device-side dense "
            "steps (Gershgorin, symmetry check, energy); one B200",
}
if args.reference:
    ref, rsec = run(0.0)
    line["reference_energy_tau0"] = ref.energy
    line["tau0_seconds"] = rsec
    line["delta_e_rel"] = abs(res.energy - ref.energy) / abs(ref.energy)
print(json.dumps(line), flush=True)
