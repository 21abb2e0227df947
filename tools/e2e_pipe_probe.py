"""Timeline of the pipelined e2e step (bench.py e2e leg): host marks per call
and device times per multiply, to see what the copy engines leave exposed."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import workloads

n, leaf = 4096, 64
taus = [1e-4, 1e-6, 1e-8, 1e-10]
a = workloads.exponential_decay(n, 0.95, 0, symmetric=True)
pins = [torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy() for _ in range(2)]
for p in pins:
    p[...] = a
G = (n // leaf) ** 2
bufs = [torch.empty((G, leaf, leaf), dtype=torch.float64, pin_memory=True).numpy() for _ in taus]
pend = [None] * 4
nxt = None
T = 12
for it in range(T):
    m = [time.perf_counter()]
    at = nxt if nxt is not None else sp.from_dense(pins[it % 2], leaf_size=leaf, wait=False)
    nxt = sp.from_dense(pins[(it + 1) % 2], leaf_size=leaf, wait=False) if it + 1 < T else None
    m.append(time.perf_counter())
    dts = []
    for q, tau in enumerate(taus):
        c, st, det = sp.spamm_detailed(at, at, sp.SpammConfig(tau=tau))
        m.append(time.perf_counter())
        dts.append((det.ms_total, det.ms_cull, det.ms_gemm, det.ms_ctree))
        if pend[q] is not None:
            pend[q].wait()
        m.append(time.perf_counter())
        pend[q] = c.nonzero_blocks(out=bufs[q], wait=False)
        c._pyramid()
        m.append(time.perf_counter())
        del c
    del at
    m.append(time.perf_counter())
    if it >= 4:
        d = np.diff(m) * 1e3
        print("step %.3f | prefetch-issue %.3f | (spamm wait issue) x4: %s | del %.3f" % (
            (m[-1] - m[0]) * 1e3, d[0], " ".join("(%.3f %.3f %.3f)" % tuple(d[1 + 3 * q:4 + 3 * q]) for q in range(4)), d[-1]))
        print("    device (total cull gemm ctree):", " ".join("(%.3f %.3f %.3f %.3f)" % x for x in dts))
for p in pend:
    p.wait()
