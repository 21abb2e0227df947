"""The CPU oracle (oracle/spamm_oracle.c) against the reference's own outputs.

tests/golden/*.npz were produced by running the real reference package
(tests/golden/make_golden.py).  The oracle must reproduce every artefact:
pyramids, retained triples, boxes and integer stats exactly, the omitted
budget bit-for-bit (numpy pairwise summation), and C bit-for-bit (its leaf
GEMM is the same sequential FMA chain the reference's BLAS used here).
"""

import numpy as np
import pytest

from oracle import oracle
from tests import golden_cases as gc

ALL = gc.case_names()


def _bits(x):
    return np.ascontiguousarray(x).view(np.uint8)


@pytest.mark.parametrize("name", ALL)
def test_oracle_matches_reference(name):
    meta, z, a, b = gc.load(name)
    dt = np.float32 if meta["dtype"] == "float32" else np.float64
    r = oracle.spamm(a, a if meta["same_operand"] else b, meta["leaf"], meta["tau"], dtype=dt,
                     tier_tau_decay=meta["tier_tau_decay"])
    assert np.array_equal(_bits(r["nsq_a"]), _bits(z["nsq_a"]))
    assert np.array_equal(r["occ_a"], z["occ_a"])
    assert np.array_equal(_bits(r["nsq_b"]), _bits(z["nsq_b"]))
    assert np.array_equal(r["triples"], z["triples"].astype(np.int32))
    assert np.array_equal(r["boxes"], z["boxes"])
    g = meta["stats"]
    for k in ("leaf_matmuls", "pruned_calls", "max_depth_reached", "pruned_volume",
              "empty_skip_volume"):
        assert r["stats"][k] == g[k], k
    assert r["stats"]["omitted_budget"].hex() == g["omitted_budget_hex"]
    if "c_padded" in z:
        assert np.array_equal(_bits(r["c_padded"]), _bits(z["c_padded"]))
    else:
        L = meta["leaf"]
        for (i, j), blk in zip(z["c_sample_ij"], z["c_sample"]):
            assert np.array_equal(_bits(r["c_padded"][i * L:(i + 1) * L, j * L:(j + 1) * L]),
                                  _bits(blk))
    assert np.array_equal(r["occ_c"], z["occ_c"])
    assert np.array_equal(_bits(r["nsq_c"]), _bits(z["nsq_c"]))
    # tiling of the index cube (test_acceptance.py:83-100 analogue)
    vol = (r["stats"]["leaf_matmuls"] * meta["leaf"] ** 3 + r["stats"]["pruned_volume"]
           + r["stats"]["empty_skip_volume"])
    assert vol == meta["padded_dim"] ** 3


def test_row_shards_sum_to_whole():
    """The multi-GPU ownership rule: disjoint C block-row shards reproduce the
    unsharded traversal (integers exactly, triples concatenated in order)."""
    meta, z, a, b = gc.load("c1")
    leaf = meta["leaf"]
    pa, pb = oracle.pad(a, leaf), oracle.pad(b, leaf)
    N = pa.shape[0]
    d = oracle.depth_for(N, leaf)
    na, oa = oracle.build_pyramid(pa, leaf)
    nb, ob = oracle.build_pyramid(pb, leaf)
    full, trip, boxes, _ = oracle.cull(na, oa, nb, ob, d, N, meta["tau"])
    for cuts in ([0, 16, 32], [0, 5, 11, 30, 32], [0, 1, 2, 3, 32]):
        tot = dict.fromkeys(full, 0)
        parts, nbox = [], 0
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            st, t, bx, _ = oracle.cull(na, oa, nb, ob, d, N, meta["tau"], rows=(lo, hi))
            for k, v in st.items():
                tot[k] = max(tot[k], v) if k == "max_depth_reached" else tot[k] + v
            parts.append(t)
            nbox += len(bx)
            assert np.all((t[:, 0] >= lo) & (t[:, 0] < hi))
        for k in ("leaf_matmuls", "pruned_calls", "pruned_volume", "empty_skip_volume",
                  "max_depth_reached"):
            assert tot[k] == full[k], (k, cuts)
        assert abs(tot["omitted_budget"] - full["omitted_budget"]) <= 1e-12 * full["omitted_budget"]
        assert np.array_equal(np.concatenate(parts), trip)
        assert nbox == len(boxes)
