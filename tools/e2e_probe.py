"""Where the e2e step's time goes: H2D/D2H bandwidths, from_dense, spamm,
pyramid reads, and the overlapped loop's per-phase host timestamps."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import workloads

n, leaf = 4096, 64
taus = [1e-4, 1e-6, 1e-8, 1e-10]
a = workloads.exponential_decay(n, 0.95, 0, symmetric=True)
if a is None:
    d = np.abs(np.subtract.outer(np.arange(n), np.arange(n))).astype(np.float64)
    u = np.random.default_rng(0).uniform(-1, 1, (n, n)) * np.power(0.95, d)
    a = 0.5 * (u + u.T)
pin = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
pin.numpy()[...] = a
dev = torch.empty((n, n), dtype=torch.float64, device="cuda")
for _ in range(3):
    dev.copy_(pin, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    dev.copy_(pin, non_blocking=True)
torch.cuda.synchronize()
h2d = (time.perf_counter() - t) / 10
print(f"H2D 134MB pinned: {h2d*1e3:.3f} ms = {n*n*8/h2d/1e9:.1f} GB/s")
t = time.perf_counter()
for _ in range(10):
    pin.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
d2h = (time.perf_counter() - t) / 10
print(f"D2H 134MB pinned: {d2h*1e3:.3f} ms = {n*n*8/d2h/1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
pin2 = torch.empty_like(pin, pin_memory=True)
dev2 = torch.empty_like(dev)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1):
        dev.copy_(pin, non_blocking=True)
    with torch.cuda.stream(s2):
        pin2.copy_(dev2, non_blocking=True)
torch.cuda.synchronize()
dup = (time.perf_counter() - t) / 10
print(f"H2D || D2H 134MB each: {dup*1e3:.3f} ms (duplex {2*n*n*8/dup/1e9:.1f} GB/s)")

G = (n // leaf) ** 2
bufs = [torch.empty((G, leaf, leaf), dtype=torch.float64, pin_memory=True).numpy() for _ in taus]
pend = [None] * 4
for it in range(8):
    marks = [time.perf_counter()]
    dts = []
    at = sp.from_dense(pin.numpy(), leaf_size=leaf)
    marks.append(time.perf_counter())
    for q, tau in enumerate(taus):
        c, st, det = sp.spamm_detailed(at, at, sp.SpammConfig(tau=tau))
        dts.append((det.ms_total, det.ms_cull, det.ms_gemm, det.ms_ctree))
        marks.append(time.perf_counter())
        if pend[q] is not None:
            pend[q].wait()
        marks.append(time.perf_counter())
        pend[q] = c.nonzero_blocks(out=bufs[q], wait=False)
        c._pyramid()
        marks.append(time.perf_counter())
        del c
    del at
    if it >= 5:
        dt = np.diff(marks) * 1e3
        print("step %.3f ms: from_dense %.3f | per tau (spamm, wait_prev, issue+pyr): %s" % (
            (marks[-1] - marks[0]) * 1e3, dt[0],
            " ".join("(%.3f %.3f %.3f)" % tuple(dt[1 + 3 * q:4 + 3 * q]) for q in range(4))))
        print("   device (total cull gemm ctree):", " ".join("(%.3f %.3f %.3f %.3f)" % x for x in dts))
for p in pend:
    p.wait()

print("synchronous reads:")
for it in range(6):
    at = sp.from_dense(pin.numpy(), leaf_size=leaf)
    dts = []
    t0 = time.perf_counter()
    for q, tau in enumerate(taus):
        c, st, det = sp.spamm_detailed(at, at, sp.SpammConfig(tau=tau))
        dts.append((det.ms_total, det.ms_cull, det.ms_gemm, det.ms_ctree))
        c.nonzero_blocks(out=bufs[q])
    if it >= 3:
        print("   %.3f ms device:" % ((time.perf_counter() - t0) * 1e3), " ".join("(%.3f %.3f %.3f %.3f)" % x for x in dts))

print("async issue + immediate wait:")
for it in range(6):
    at = sp.from_dense(pin.numpy(), leaf_size=leaf)
    dts = []
    t0 = time.perf_counter()
    for q, tau in enumerate(taus):
        c, st, det = sp.spamm_detailed(at, at, sp.SpammConfig(tau=tau))
        dts.append((det.ms_total, det.ms_cull, det.ms_gemm, det.ms_ctree))
        c.nonzero_blocks(out=bufs[q], wait=False).wait()
    if it >= 3:
        print("   %.3f ms device:" % ((time.perf_counter() - t0) * 1e3), " ".join("(%.3f %.3f %.3f %.3f)" % x for x in dts))

print("sync reads + unrelated torch D2H (32 MB) in flight during each spamm:")
src = torch.empty(4 * 1024 * 1024, dtype=torch.float64, device="cuda")
dst = torch.empty(4 * 1024 * 1024, dtype=torch.float64, pin_memory=True)
side = torch.cuda.Stream()
for it in range(6):
    at = sp.from_dense(pin.numpy(), leaf_size=leaf)
    dts = []
    t0 = time.perf_counter()
    for q, tau in enumerate(taus):
        with torch.cuda.stream(side):
            dst.copy_(src, non_blocking=True)
        c, st, det = sp.spamm_detailed(at, at, sp.SpammConfig(tau=tau))
        dts.append((det.ms_total, det.ms_cull, det.ms_gemm, det.ms_ctree))
        c.nonzero_blocks(out=bufs[q])
    if it >= 3:
        print("   %.3f ms device:" % ((time.perf_counter() - t0) * 1e3), " ".join("(%.3f %.3f %.3f %.3f)" % x for x in dts))
print("sync reads + unrelated torch H2D (32 MB) in flight during each spamm:")
for it in range(6):
    at = sp.from_dense(pin.numpy(), leaf_size=leaf)
    dts = []
    t0 = time.perf_counter()
    for q, tau in enumerate(taus):
        with torch.cuda.stream(side):
            src.copy_(dst, non_blocking=True)
        c, st, det = sp.spamm_detailed(at, at, sp.SpammConfig(tau=tau))
        dts.append((det.ms_total, det.ms_cull, det.ms_gemm, det.ms_ctree))
        c.nonzero_blocks(out=bufs[q])
    if it >= 3:
        print("   %.3f ms device:" % ((time.perf_counter() - t0) * 1e3), " ".join("(%.3f %.3f %.3f %.3f)" % x for x in dts))


print("async, one shared 40 MB pinned buffer (wait before reuse):")
one = torch.empty((1200, leaf, leaf), dtype=torch.float64, pin_memory=True).numpy()
prev = None
for it in range(8):
    marks = [time.perf_counter()]
    at = sp.from_dense(pin.numpy(), leaf_size=leaf)
    marks.append(time.perf_counter())
    dts = []
    for q, tau in enumerate(taus):
        c, st, det = sp.spamm_detailed(at, at, sp.SpammConfig(tau=tau))
        dts.append((det.ms_total, det.ms_cull, det.ms_gemm, det.ms_ctree))
        if prev is not None:
            prev.wait()
        prev = c.nonzero_blocks(out=one, wait=False)
        del c
    marks.append(time.perf_counter())
    if it >= 5:
        print("   step %.3f ms (from_dense %.3f) device:" % ((marks[-1] - marks[0]) * 1e3, (marks[1]-marks[0])*1e3), " ".join("(%.3f %.3f %.3f %.3f)" % x for x in dts))
prev.wait()
