"""Golden fixtures for the matched-error threshold search, produced by running
the REAL reference package (build container only):

    SPAMM_REF=/root/reference/pkg/src python tests/golden/make_match_golden.py

The cases are those of the reference's acceptance test
(pkg/tests/test_acceptance.py:139-186): gapped chain n = 256 at targets 1e-6
and 1e-8, gapless at 1e-5, in-multiply pruning and drop-then-multiply, 16
bisection steps.  The searches visit coarse thresholds whose iterates diverge
(NaN traces), so they pin the driver's behaviour there too.  Floats are stored
as hex strings (bit for bit).
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("SPAMM_REF", "/root/reference/pkg/src"))
sys.dont_write_bytecode = True

from spamm import purification as P  # noqa: E402  (the reference)
from spamm.generators import ModelHamiltonian, gen_model_hamiltonian  # noqa: E402

CASES = (("gapped", 1e-6), ("gapped", 1e-8), ("gapless", 1e-5))


def main():
    out = {}
    exact = {}
    for kind, target in CASES:
        n = 256
        f = gen_model_hamiltonian(ModelHamiltonian(n=n, kind=kind))
        if kind not in exact:
            exact[kind] = P.purify(f, n // 2, P.SpammMode(0.0)).energy
        for name, mode in (("spamm", P.SpammMode(0.0)), ("drop", P.DroppingMode(0.0))):
            r = P.match_error_threshold(f, n // 2, target, mode, max_steps=16,
                                        reference_energy=exact[kind])
            out[f"{kind}_{target:.0e}_{name}"] = {
                "kind": kind, "target": target, "mode": name,
                "exact_energy": float(exact[kind]).hex(),
                "tau": float(r.tau).hex(), "delta_e_rel": float(r.delta_e_rel).hex(),
                "converged": bool(r.converged), "hit_boundary": bool(r.hit_boundary),
                "evaluations": int(r.evaluations),
                "energy": float(r.result.energy).hex(),
                "total_leaf_matmuls": int(r.result.total_leaf_matmuls),
                "step_leaf_matmuls": [int(c) for c in r.result.step_leaf_matmuls],
            }
            print(kind, target, name, r.tau, r.delta_e_rel, r.converged, r.evaluations,
                  r.result.avg_leaf_matmuls, flush=True)
    with open(os.path.join(HERE, "match_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
