"""Golden fixtures for the box log, the MatrixMarket writer and the matrix
generators, produced by running the REAL reference package (build container
only):

    SPAMM_REF=/root/reference/pkg/src python tests/golden/make_io_golden.py

Writes into tests/golden/io/:
  boxlog_exp128.txt   write_box_log of spamm(gen_exponential(128, 1.0),
                      gen_exponential(128, 2.0), tau=1e-6) (the reference's
                      own box-log test case) -- plus boxlog_l16_b4.txt for a
                      deeper tree (n = 512, leaf 4, tau = 1e-7)
  mm_array.mtx, mm_coord.mtx   write_matrix_market of a small matrix with
                      negative zero, subnormal, huge and integral values
  io_golden.npz       that matrix; the dense matrices of gen_exponential,
                      gen_algebraic and gen_model_hamiltonian (padded arrays
                      and norm pyramids) for a few sizes/parameters
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "io")
sys.path.insert(0, os.environ.get("SPAMM_REF", "/root/reference/pkg/src"))
sys.dont_write_bytecode = True

from spamm import generators as G  # noqa: E402  (the reference)
from spamm import matrixmarket as MM  # noqa: E402
from spamm import multiply as M  # noqa: E402

GEN_CASES = [
    ("exp_n100_a0.3_b4", lambda: G.gen_exponential(100, 0.3)),
    ("exp_n257_a1.7_b8", lambda: G.gen_exponential(257, 1.7, leaf_size=8)),
    ("exp_n64_a0.05_b16", lambda: G.gen_exponential(64, 0.05, leaf_size=16)),
    ("alg_n100_p1.5_b4", lambda: G.gen_algebraic(100, 1.5)),
    ("alg_n130_p0.7_b2", lambda: G.gen_algebraic(130, 0.7, leaf_size=2)),
    ("alg_n64_p3_b8", lambda: G.gen_algebraic(64, 3, leaf_size=8)),
    ("ham_gapped_n96_b4", lambda: G.gen_model_hamiltonian(G.ModelHamiltonian(96))),
    ("ham_gapped_n37_g0.3_t-1.25_b4",
     lambda: G.gen_model_hamiltonian(G.ModelHamiltonian(37, gap=0.3, hopping=-1.25))),
    ("ham_gapless_n50_b8",
     lambda: G.gen_model_hamiltonian(G.ModelHamiltonian(50, kind="gapless"), leaf_size=8)),
]


def pyramid(t):
    return np.concatenate([np.asarray(x, dtype=np.float64).ravel() for x in t._norm_sq])


def main():
    os.makedirs(OUT, exist_ok=True)
    out = {}
    a = G.gen_exponential(128, 1.0)
    b = G.gen_exponential(128, 2.0)
    _, st = M.spamm(a, b, M.SpammConfig(tau=1e-6, collect_boxes=True))
    M.write_box_log(st.boxes, os.path.join(OUT, "boxlog_exp128.txt"), a.padded_dim)
    out["boxlog_exp128_n"] = np.int64(len(st.boxes))

    a = G.gen_exponential(512, 0.4)
    b = G.gen_algebraic(512, 2.5)
    _, st = M.spamm(a, b, M.SpammConfig(tau=1e-7, collect_boxes=True))
    M.write_box_log(st.boxes, os.path.join(OUT, "boxlog_l16_b4.txt"), a.padded_dim)
    out["boxlog_l16_b4_n"] = np.int64(len(st.boxes))

    rng = np.random.default_rng(7)
    m = rng.standard_normal((7, 5))
    m[0, 0] = -0.0
    m[1, 2] = 5e-324
    m[2, 3] = 1.7976931348623157e308
    m[3, 1] = 3.0
    m[4, :] = 0.0
    m[:, 4] = 0.0
    m[5, 4] = 0.1
    out["mm_matrix"] = m
    MM.write_matrix_market(m, os.path.join(OUT, "mm_array.mtx"), fmt="array")
    MM.write_matrix_market(m, os.path.join(OUT, "mm_coord.mtx"), fmt="coordinate")

    for name, make in GEN_CASES:
        t = make()
        out[f"gen_{name}_padded"] = np.asarray(t._padded)
        out[f"gen_{name}_nsq"] = pyramid(t)
    np.savez_compressed(os.path.join(OUT, "io_golden.npz"), **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
