"""Determinism stress: many multiplies over interleaved geometries, each
compared bit for bit with the first result of the same configuration (C's
storage hash, C's pyramid, integer stats, budget bits).  Geometries whose
group sets differ call after call (different tau, operands, leaf sizes, row
shards, dense and tiered traversals), so stale scratch from the previous call
cannot pass for the current one.

    python tools/stress.py [--rounds R] [--procs P] [--seed S] [--big]

--procs P runs P processes on the same GPU at once (their kernels time-slice,
which perturbs every kernel's timing).  --big adds an n = 16384 case (tiered
traversal, regular C tree).  Prints one JSON line per process; exit status 1
on any mismatch."""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _configs(big):
    from paper_1011_3534_b200 import workloads

    a1, b1, l1, t1 = workloads.make_config("c1")
    a2, _, l2, t2 = workloads.make_config("c2")
    a3, b3, l3, t3 = workloads.make_config("c3_l3")
    cfgs = [("c1", a1, b1, l1, t1[0], None)]
    for t in t2:
        cfgs.append((f"c2_tau{t:g}", a2, a2, l2, t, None))
    cfgs.append(("c2_rows_lo", a2, a2, l2, t2[1], (0, 23)))
    cfgs.append(("c2_rows_hi", a2, a2, l2, t2[3], (23, 64)))
    cfgs.append(("c3_l3_tau1e-6", a3, b3, l3, t3[0], None))
    cfgs.append(("c2_leaf32", a2, a2, 32, 1e-8, None))
    if big:
        a5 = workloads.exponential_decay(16384, 0.98, 0, symmetric=True)
        cfgs.append(("c5_proxy16k", a5, a5, 64, 1e-8, None))
    return cfgs


def _digest(c, st):
    import torch

    from paper_1011_3534_b200 import distributed as spd

    cs = spd.tree_storage(c)  # (a lazy product is zero-filled where empty)
    w = torch.arange(1, cs.numel() + 1, device=cs.device, dtype=torch.int64).view(cs.shape)
    h = int((cs.contiguous().view(torch.int64) * w).sum().item()) if cs.dtype == torch.float64 else \
        int((cs.contiguous().view(torch.int32).to(torch.int64) * w).sum().item())
    pyr = c._pyramid()
    ph = hash(pyr[2].tobytes()) ^ hash(pyr[3].tobytes())
    return (h, ph, st.leaf_matmuls, st.pruned_calls, st.pruned_volume, st.empty_skip_volume,
            float(st.omitted_budget).hex())


def _purify_digest(h, sweeps):
    import paper_1011_3534_b200 as sp
    from paper_1011_3534_b200 import purification as P

    res = P.purify(sp.from_dense(h, leaf_size=64), h.shape[0] // 2, P.SpammMode(1e-7),
                   max_iter=sweeps, reference_energy=0.0)
    st = type("S", (), dict(leaf_matmuls=tuple(res.step_leaf_matmuls), pruned_calls=0,
                            pruned_volume=0, empty_skip_volume=0, omitted_budget=res.energy))
    return (tuple(float(t).hex() for t in res.trace_history),) + _digest(res.density, st)


def run(rounds, seed, big, purify=0):
    import paper_1011_3534_b200 as sp

    sp.set_device(0)
    trees = {}
    cfgs = _configs(big)
    first = {}
    bad = []
    rng = np.random.default_rng(seed)
    n_mult = 0
    if purify:
        from paper_1011_3534_b200 import workloads
        cfgs.append(("purify_L16", workloads.cubic_lattice_hamiltonian(16), None, 64, purify, None))
    t0 = time.time()
    for r in range(rounds + 1):
        order = rng.permutation(len(cfgs)) if r else np.arange(len(cfgs))
        for q in order:
            name, a, b, leaf, tau, rows = cfgs[q]
            if name.startswith("purify"):
                d = _purify_digest(a, tau)
                if r == 0:
                    first[name] = d
                elif d != first[name]:
                    bad.append(dict(round=r, config=name, got=str(d)[:400], want=str(first[name])[:400]))
                continue
            key = (id(a), leaf)
            if key not in trees:
                trees[key] = sp.from_dense(a, leaf_size=leaf)
            kb = (id(b), leaf)
            if kb not in trees:
                trees[kb] = sp.from_dense(b, leaf_size=leaf)
            A, B = trees[key], trees[kb]
            c, st, _ = sp.spamm_detailed(A, B, sp.SpammConfig(tau=tau), rows=rows)
            d = _digest(c, st)
            n_mult += 1
            if r == 0:
                first[name] = d
            elif d != first[name]:
                bad.append(dict(round=r, config=name, got=str(d), want=str(first[name])))
            del c
    return dict(pid=os.getpid(), rounds=rounds, multiplies=n_mult, mismatches=len(bad),
                first_mismatches=bad[:5], seconds=round(time.time() - t0, 1))


def _child(args):
    res = run(args.rounds, args.seed, args.big, args.purify)
    print(json.dumps(res), flush=True)
    return 0 if res["mismatches"] == 0 else 1


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=25)
    ap.add_argument("--procs", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--purify", type=int, default=0, help="add a TC2 purification of N sweeps")
    args = ap.parse_args()
    if args.procs <= 1 or args.child:
        sys.exit(_child(args))
    import subprocess

    procs = [subprocess.Popen([sys.executable, __file__, "--child", "--rounds", str(args.rounds),
                               "--seed", str(args.seed + p), "--purify", str(args.purify)]
                              + (["--big"] if args.big else []))
             for p in range(args.procs)]
    rc = max(p.wait() for p in procs)
    sys.exit(rc)
