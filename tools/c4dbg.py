import sys; sys.path.insert(0,'.')
import numpy as np, torch
import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import purification as P, workloads
L = int(sys.argv[1]); n = L**3
h = workloads.cubic_lattice_hamiltonian_device(L, "cuda:0")
f = sp.from_device_pointer(h.data_ptr(), n, leaf_size=64)
for tau in (1e-7, 0.0):
    res = P.purify(f, n//2, P.SpammMode(tau), max_iter=30, reference_energy=float('nan'))
    print(L, tau, P.HOST_DENSE_MAX, res.energy, res.trace_history[:4], res.trace_history[-3:], res.step_leaf_matmuls[-3:], flush=True)
