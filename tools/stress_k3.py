"""Debug: repeat one multiply with deep merge stacks (dense operands, tau = 0:
64 products per C block) and compare C bit for bit with the first result.

    python tools/stress_k3.py [--reps R] [--procs P] [--n 4096]"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(a):
    import numpy as np
    import torch

    import paper_1011_3534_b200 as sp
    from paper_1011_3534_b200 import distributed as spd

    sp.set_device(0)
    rng = np.random.default_rng(1)
    A = sp.from_dense(rng.standard_normal((a.n, a.n)), leaf_size=64)
    ref = None
    ev = []
    for r in range(a.reps):
        c, st = sp.spamm(A, A, sp.SpammConfig(tau=a.tau))
        cs = spd.tree_storage(c).view(torch.int64)
        if ref is None:
            ref = cs.clone()
        elif not torch.equal(cs, ref):
            d = cs != ref
            idx = d.nonzero()
            blocks = sorted({(int(i) // 64, int(j) // 64) for i, j in idx[:4096].tolist()})
            bi, bj = blocks[0]
            sub = d[bi * 64:(bi + 1) * 64, bj * 64:(bj + 1) * 64]
            ev.append(dict(rep=r, n_diff=int(d.sum()), blocks=blocks[:8],
                           rows=sub.any(1).nonzero().flatten().tolist(),
                           cols=sub.any(0).nonzero().flatten().tolist()))
        del c
    print(json.dumps(dict(pid=os.getpid(), reps=a.reps, n_events=len(ev), events=ev[:6])), flush=True)
    return 1 if ev else 0


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=300)
    ap.add_argument("--procs", type=int, default=1)
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--tau", type=float, default=0.0)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.procs <= 1 or a.child:
        sys.exit(main(a))
    ps = [subprocess.Popen([sys.executable, __file__, "--child", "--reps", str(a.reps), "--n", str(a.n),
                            "--tau", str(a.tau)]) for _ in range(a.procs)]
    sys.exit(max(p.wait() for p in ps))
