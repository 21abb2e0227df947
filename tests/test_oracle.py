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


def test_oracle_pieces_reassemble_the_whole_multiply():
    """oracle.leaf_norms + pyramid_from_leaves rebuild C's pyramid and
    oracle.group_product rebuilds every C block from gathered operand blocks
    (the pieces the full-size GPU checks use) -- bit for bit vs the dense
    oracle on config 1."""
    from oracle import oracle
    from paper_1011_3534_b200 import workloads

    a, b, leaf, taus = workloads.make_config("c1")
    r = oracle.spamm(a, b, leaf, taus[0])
    N, depth = r["N"], r["depth"]
    nb = N // leaf
    blk = r["c_padded"].reshape(nb, leaf, nb, leaf).swapaxes(1, 2).reshape(-1, leaf, leaf)
    nsq, occ = oracle.pyramid_from_leaves(*oracle.leaf_norms(blk), depth)
    assert np.array_equal(nsq.view(np.uint64), r["nsq_c"].view(np.uint64))
    assert np.array_equal(occ, r["occ_c"])
    t, pa, pb = r["triples"], r["a_padded"], r["b_padded"]
    gid = t[:, 0].astype(np.int64) * nb + t[:, 1]
    starts = np.flatnonzero(np.r_[True, gid[1:] != gid[:-1]])
    for s0, s1 in zip(starts, np.r_[starts[1:], len(t)]):
        i, j, ks = t[s0, 0], t[s0, 1], t[s0:s1, 2]
        A = np.stack([pa[i * leaf:(i + 1) * leaf, k * leaf:(k + 1) * leaf] for k in ks])
        B = np.stack([pb[k * leaf:(k + 1) * leaf, j * leaf:(j + 1) * leaf] for k in ks])
        got = oracle.group_product(A, B, ks, depth)
        want = r["c_padded"][i * leaf:(i + 1) * leaf, j * leaf:(j + 1) * leaf]
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (i, j)
