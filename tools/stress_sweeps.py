"""Debug: repeat a TC2 run sweep by sweep and compare every X^2 and next
iterate with the first run's (kept on the device); report the first sweep
whose input was identical but whose product (or update) differs, and how.

    python tools/stress_sweeps.py [--runs R] [--procs P] [--L 16] [--sweeps 12]"""

import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(args):
    import torch

    import paper_1011_3534_b200 as sp
    from paper_1011_3534_b200 import distributed as spd
    from paper_1011_3534_b200 import purification as P
    from paper_1011_3534_b200 import workloads
    from paper_1011_3534_b200.quadtree import tc2_update, trace

    sp.set_device(0)
    h = workloads.cubic_lattice_hamiltonian(args.L)
    n = h.shape[0]
    f = sp.from_dense(h, leaf_size=64)
    ref = None
    events = []
    for run in range(args.runs):
        x = P.tc2_initial_guess(f)
        rec = []
        for s in range(args.sweeps):
            xs = spd.tree_storage(x).clone()
            torch.cuda.synchronize()  # (the clone must finish before the library frees x)
            tr = trace(x)
            x2, st, det = sp.spamm_detailed(x, x, sp.SpammConfig(tau=args.tau), keep_triples=True)
            x2s = spd.tree_storage(x2).clone()
            torch.cuda.synchronize()
            mk = tr < n // 2
            y, _, _, dn, en = tc2_update(x, x2, make_y=mk)
            ys = spd.tree_storage(y).clone() if mk else None
            torch.cuda.synchronize()
            rec.append((xs, x2s, ys, st.leaf_matmuls, det.triples.copy(), dn, en))
            x = x2 if not mk else y
        if ref is None:
            ref = rec
            continue
        for s in range(args.sweeps):
            xs, x2s, ys, cnt, tri, dn, en = rec[s]
            rxs, rx2s, rys, rcnt, rtri, rdn, ren = ref[s]
            same_in = torch.equal(xs.view(torch.int64), rxs.view(torch.int64))
            same_x2 = torch.equal(x2s.view(torch.int64), rx2s.view(torch.int64))
            same_y = ys is None or torch.equal(ys.view(torch.int64), rys.view(torch.int64))
            if same_in and same_x2 and same_y and dn == rdn and en == ren:
                continue
            ev = dict(run=run, sweep=s, same_input=same_in, same_x2=same_x2, same_y=same_y,
                      same_triples=bool(np.array_equal(tri, rtri)), count=cnt, ref_count=rcnt,
                      dn_same=dn == rdn, en_same=en == ren)
            if same_in and not same_x2:
                d = (x2s.view(torch.int64) != rx2s.view(torch.int64))
                idx = d.nonzero()
                blocks = sorted({(int(r) // 64, int(c) // 64) for r, c in idx[:20000].tolist()})
                diff = (x2s - rx2s).abs()
                ev.update(n_diff=int(d.sum()), blocks=blocks[:20], n_blocks=len(blocks),
                          max_abs=float(diff.max()), max_rel=float((diff / rx2s.abs().clamp_min(1e-300)).max()))
                # per differing block: rows/cols pattern
                if blocks:
                    bi, bj = blocks[0]
                    sub = d[bi * 64:(bi + 1) * 64, bj * 64:(bj + 1) * 64]
                    ev.update(first_block_rows=sub.any(1).nonzero().flatten().tolist()[:64],
                              first_block_cols=sub.any(0).nonzero().flatten().tolist()[:64])
                    ks = tri[(tri[:, 0] == bi) & (tri[:, 1] == bj)][:, 2].tolist()
                    ev.update(first_block_ks=ks)
            events.append(ev)
            break  # later sweeps follow from this one
    print(json.dumps(dict(pid=os.getpid(), runs=args.runs, events=events[:10], n_events=len(events))),
          flush=True)
    return 1 if events else 0


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=20)
    ap.add_argument("--procs", type=int, default=1)
    ap.add_argument("--L", type=int, default=16)
    ap.add_argument("--sweeps", type=int, default=12)
    ap.add_argument("--tau", type=float, default=1e-7)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.procs <= 1 or a.child:
        sys.exit(main(a))
    ps = [subprocess.Popen([sys.executable, __file__, "--child", "--runs", str(a.runs), "--L", str(a.L),
                            "--sweeps", str(a.sweeps), "--tau", str(a.tau)]) for _ in range(a.procs)]
    sys.exit(max(p.wait() for p in ps))
