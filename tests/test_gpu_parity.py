"""GPU parity: the CUDA path through the C ABI vs the reference's outputs.

Every golden case (tests/golden, produced by the real reference) is rerun on
the B200 and compared:
* norm / occupancy pyramids of A, B and C: bit-exact
* retained leaf-triple set and pruned boxes (in reference order): exact
* ProductStats integers: exact; omitted_budget: bit-exact (numpy pairwise)
* C: bit-exact vs the reference (DMMA == the BLAS FMA chain, same merge
  tree) -- whole for small cases; for the large ones every nonzero block
  through a 64-bit hash of its bits plus eight blocks byte for byte; the
  contract bar, 1e-12 relative Frobenius, is asserted as well.
"""

import numpy as np
import pytest

import paper_1011_3534_b200 as sp
from tests import golden_cases as gc

pytestmark = pytest.mark.gpu

SMALL = gc.case_names(max_n=1024)
LARGE = [n for n in gc.case_names() if n not in SMALL]


def _run(name, traversal="auto"):
    meta, z, a_d, b_d = gc.load(name)
    leaf = meta["leaf"]
    a = sp.from_dense(a_d, leaf_size=leaf, dtype=a_d.dtype)
    b = a if meta["same_operand"] else sp.from_dense(b_d, leaf_size=leaf, dtype=b_d.dtype)
    cfg = sp.SpammConfig(tau=meta["tau"], collect_boxes=True,
                         tier_tau_decay=meta["tier_tau_decay"])
    c, st, det = sp.spamm_detailed(a, b, cfg, keep_triples=True, traversal=traversal)
    return meta, z, a, b, c, st, det


def _pyr(t):
    return t._pyramid()[2], t._pyramid()[3]


def _check(name, traversal="auto"):
    meta, z, a, b, c, st, det = _run(name, traversal)
    na, oa = _pyr(a)
    assert np.array_equal(na.view(np.uint64), z["nsq_a"].view(np.uint64)), "A norms"
    assert np.array_equal(oa, z["occ_a"]), "A occupancy"
    nb_, ob = _pyr(b)
    assert np.array_equal(nb_.view(np.uint64), z["nsq_b"].view(np.uint64)), "B norms"
    assert np.array_equal(ob, z["occ_b"]), "B occupancy"
    g = meta["stats"]
    assert st.leaf_matmuls == g["leaf_matmuls"]
    assert st.pruned_calls == g["pruned_calls"]
    assert st.max_depth_reached == g["max_depth_reached"]
    assert st.pruned_volume == g["pruned_volume"]
    assert st.empty_skip_volume == g["empty_skip_volume"]
    assert st.omitted_budget == g["omitted_budget"], (st.omitted_budget, g["omitted_budget"])
    assert np.array_equal(det.triples, z["triples"].astype(np.int32)), "retained triples"
    boxes = np.array([[bx.i_lo, bx.j_lo, bx.k_lo, bx.edge, bx.tier] for bx in st.boxes],
                     np.int64).reshape(-1, 5)
    assert np.array_equal(boxes, z["boxes"]), "pruned boxes"
    assert st.covered_volume(meta["leaf"]) == meta["padded_dim"] ** 3
    L = meta["leaf"]
    if "c_padded" in z:
        got = c._padded
        ref = z["c_padded"]
        den = np.linalg.norm(ref.astype(np.float64)) or 1.0
        assert np.linalg.norm(got.astype(np.float64) - ref) / den <= 1e-12
        assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), "C bit-exact"
    else:
        nbk = c.block_grid
        for (i, j), blk in zip(z["c_sample_ij"], z["c_sample"]):
            mine = gc.tree_blocks(c, [int(i) * nbk + int(j)])[0]
            assert np.array_equal(mine.view(np.uint8), blk.view(np.uint8)), ("C block", i, j)
        if "c_block_ids" in z:  # every nonzero block of C, pinned by its hash
            ids, want = z["c_block_ids"], z["c_block_hash"]
            mine_ids = np.flatnonzero(np.asarray(c._leaf_nonzero).reshape(-1))
            assert np.array_equal(mine_ids, ids), "C's nonzero blocks"
            got = gc.tree_block_hashes(c, ids)
            bad = np.flatnonzero(got != want)
            assert bad.size == 0, f"{bad.size} of {len(ids)} C blocks differ, first id {ids[bad[0]]}"
    nc, oc = _pyr(c)
    assert np.array_equal(oc, z["occ_c"]), "C occupancy"
    assert np.array_equal(nc.view(np.uint64), z["nsq_c"].view(np.uint64)), "C norms"
    return meta, a, b, c


# "auto" takes the dense single-pass traversal for depth <= 6 (most golden
# cases), "tiered" the breadth-first tier kernel: both must match.
@pytest.mark.parametrize("traversal", ["auto", "tiered"])
@pytest.mark.parametrize("name", SMALL)
def test_golden_small(name, traversal):
    _check(name, traversal)


@pytest.mark.parametrize("traversal", ["auto", "tiered"])
@pytest.mark.parametrize("name", LARGE)
def test_golden_large(name, traversal):
    meta, a, b, c = _check(name, traversal)
    # SpAMM-vs-exact error equals the reference's (multiply_error)
    err, budget = sp.multiply_error(a, b, sp.SpammConfig(tau=meta["tau"]))
    assert abs(err - meta["abs_err"]) <= 1e-9 * max(meta["abs_err"], 1e-300) + 1e-15 * meta["norm_a"] * meta["norm_b"]
    assert budget == meta["budget_from_error_run"]
