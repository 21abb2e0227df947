"""Golden fixtures for the tree algebra and the TC2 purification driver,
produced by running the REAL reference package (build container only):

    SPAMM_REF=/root/reference/pkg/src python tests/golden/make_purify_golden.py

Records, per case, the reference's outputs bit for bit: padded arrays and
norm/occupancy pyramids of add / scale / filter_drop results, traces, and for
purify() the final density, trace history, per-sweep leaf multiplies, energy,
reference energy and delta_e_rel.  Inputs are small and stored alongside.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.environ.get("SPAMM_REF", "/root/reference/pkg/src"))
sys.dont_write_bytecode = True

from spamm import quadtree as Q  # noqa: E402  (the reference)
from spamm import purification as P  # noqa: E402
from spamm.generators import ModelHamiltonian, gen_model_hamiltonian  # noqa: E402

from paper_1011_3534_b200 import workloads  # noqa: E402


def pyramid(t):
    nsq = np.concatenate([np.asarray(x, dtype=np.float64).ravel() for x in t._norm_sq])
    occ = np.concatenate([np.asarray(x, dtype=np.uint8).ravel() for x in t._occupied])
    return nsq, occ


def tree_arrays(prefix, t, out):
    out[prefix + "_padded"] = np.asarray(t._padded)
    out[prefix + "_nsq"], out[prefix + "_occ"] = pyramid(t)


def algebra_inputs(dtype):
    rng = np.random.default_rng(11)
    n, leaf = 40, 8
    a = rng.uniform(-1, 1, (n, n))
    a[8:16, :] = 0.0            # empty blocks
    a[:, 24:32] = 0.0
    a[0, 0] = -0.0
    a[33, 2] = -0.0
    b = rng.uniform(-1, 1, (n, n))
    b[0:8, 8:16] = -a[0:8, 8:16]    # cancels to zero in a + b
    b[16:24, 16:24] = 0.0           # a-only block
    b[8:16, 32:40] = rng.uniform(-1, 1, (8, 8))  # b-only block (a is zero there)
    b[20, 20] = -0.0
    return a.astype(dtype), b.astype(dtype), leaf


def algebra_cases():
    out, meta = {}, {}
    for dname, dt in (("f64", np.float64), ("f32", np.float32)):
        a, b, leaf = algebra_inputs(dt)
        out[f"{dname}_a"], out[f"{dname}_b"] = a, b
        ta = Q.from_dense(a, leaf_size=leaf, dtype=dt)
        tb = Q.from_dense(b, leaf_size=leaf, dtype=dt)
        tree_arrays(f"{dname}_add", Q.add(ta, tb), out)
        tree_arrays(f"{dname}_scale_m15", Q.scale(ta, -1.5), out)
        tree_arrays(f"{dname}_scale_0", Q.scale(ta, 0.0), out)
        tree_arrays(f"{dname}_scale_third", Q.scale(tb, 1.0 / 3.0), out)
        leaf_norms = np.sqrt(np.asarray(ta._norm_sq[ta.depth], dtype=np.float64))
        occupied = leaf_norms[np.asarray(ta._leaf_nonzero)]
        tau_mid = float(np.median(occupied))
        meta[f"{dname}_tau_mid"] = tau_mid
        tree_arrays(f"{dname}_filter_mid", Q.filter_drop(ta, tau_mid), out)
        meta[f"{dname}_filter_none_is_input"] = Q.filter_drop(ta, 0.0) is ta
        meta[f"{dname}_trace_a"] = Q.trace(ta)
        meta[f"{dname}_trace_add"] = Q.trace(Q.add(ta, tb))
    return out, meta


def purify_case(name, f_dense, leaf, n_occ, mode, max_iter, out, meta):
    f = Q.from_dense(f_dense, leaf_size=leaf)
    res = P.purify(f, n_occ, mode, max_iter=max_iter)
    out[f"{name}_f"] = f_dense
    out[f"{name}_density"] = np.asarray(res.density._padded)
    meta[name] = dict(leaf=leaf, n_occ=n_occ, mode=type(mode).__name__, tau=mode.tau,
                      max_iter=max_iter, energy=res.energy, delta_e_rel=res.delta_e_rel,
                      reference_energy=res.reference_energy, trace_history=res.trace_history,
                      step_leaf_matmuls=[int(x) for x in res.step_leaf_matmuls],
                      total_leaf_matmuls=res.total_leaf_matmuls)


def main():
    out, meta = algebra_cases()
    chain = np.asarray(gen_model_hamiltonian(ModelHamiltonian(64, "gapped"), leaf_size=4)._padded)[:64, :64]
    purify_case("chain64_spamm", chain, 4, 32, P.SpammMode(1e-6), 12, out, meta)
    purify_case("chain64_drop", chain, 4, 32, P.DroppingMode(1e-4), 12, out, meta)
    lat4 = workloads.cubic_lattice_hamiltonian(4)
    purify_case("lattice4_spamm", lat4, 8, 32, P.SpammMode(1e-7), 30, out, meta)
    lat8 = workloads.cubic_lattice_hamiltonian(8)
    purify_case("lattice8_spamm", lat8, 16, 256, P.SpammMode(1e-7), 30, out, meta)
    np.savez_compressed(os.path.join(HERE, "purify_golden.npz"), **out)
    with open(os.path.join(HERE, "purify_golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("wrote", len(out), "arrays;", list(meta))


if __name__ == "__main__":
    main()
