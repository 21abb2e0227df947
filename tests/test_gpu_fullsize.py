"""Parity at BASELINE.json's full sizes, where the oracle cannot hold the
operands densely: config 5 (n = 65536, leaf 64, tau = 1e-8; f64 and the f32
variant) and config 4's first SP2 sweeps (32^3 lattice, n = 32768, leaf 64,
tau = 1e-7).

The GPU's result is checked against the CPU oracle on the same inputs through
what the oracle can hold:
* the retained leaf-triple set, the pruned boxes in reference order, every
  ProductStats integer and the budget's bits -- oracle.cull on the operand
  pyramids pulled off the device (multiply.py:178-212);
* sampled C blocks, bit for bit -- oracle.group_product on the operand blocks
  of each sampled block's retained triples (multiply.py:224-257, :119-141);
* C's whole norm / occupancy pyramid, bit for bit -- oracle.leaf_norms over
  every nonzero C block pulled off the device, then oracle.pyramid_from_leaves
  (multiply.py:220 -> quadtree.py:74-92, :126-138).
The operands themselves are pinned by their pyramids (K1 is checked bit-exact
against the reference elsewhere) -- here they are the inputs both sides share.
"""

import numpy as np
import pytest

import paper_1011_3534_b200 as sp
from oracle import oracle
from tests import golden_cases as gc

pytestmark = pytest.mark.gpu


def _pyr(t):
    return t._pyramid()[2], t._pyramid()[3]


def check_product_vs_oracle(a, b, c, st, det, tau, n_sample=64, seed=0):
    """Every check above for one device product c = spamm(a, b, tau)."""
    depth, N, nbk = a.depth, a.padded_dim, a.block_grid
    na, oa = _pyr(a)
    nb_, ob = (na, oa) if b is a else _pyr(b)
    ref, trip, boxes, tiers = oracle.cull(na, oa, nb_, ob, depth, N, tau, collect_boxes=True)
    assert st.leaf_matmuls == ref["leaf_matmuls"]
    assert np.array_equal(det.triples, trip), "retained triples"
    for k in ("pruned_calls", "pruned_volume", "empty_skip_volume", "max_depth_reached"):
        assert getattr(st, k) == ref[k], k
    assert st.omitted_budget == ref["omitted_budget"], (st.omitted_budget, ref["omitted_budget"])
    got_boxes = np.array([[x.i_lo, x.j_lo, x.k_lo, x.edge, x.tier] for x in st.boxes],
                         np.int64).reshape(-1, 5)
    assert np.array_equal(got_boxes, boxes), "pruned boxes"
    assert det.tier_candidates == tiers["candidates"]
    assert det.tier_survivors == tiers["survivors"]
    # the product's nonzero blocks lie within the retained (i, j) groups (a
    # group whose products cancel exactly -- sparse blocks with disjoint
    # patterns -- leaves an all-zero, unoccupied block: quadtree.py:126)
    gid = trip[:, 0].astype(np.int64) * nbk + trip[:, 1]
    starts = np.flatnonzero(np.r_[True, gid[1:] != gid[:-1]])
    groups = gid[starts]
    occ_c = np.asarray(c._leaf_nonzero).reshape(-1)
    assert np.isin(np.flatnonzero(occ_c), groups).all(), "C's nonzero blocks"
    assert np.count_nonzero(occ_c) <= len(groups)
    # sampled C blocks, bit for bit
    rng = np.random.default_rng(seed)
    ends = np.r_[starts[1:], len(gid)]
    order = np.argsort(ends - starts)  # always include the largest and smallest groups
    pick = np.unique(np.r_[order[:2], order[-2:],
                           rng.choice(len(groups), size=min(n_sample, len(groups)), replace=False)])
    for g in pick:
        s0, s1 = starts[g], ends[g]
        i, j = int(trip[s0, 0]), int(trip[s0, 1])
        ks = trip[s0:s1, 2]
        ab = gc.tree_blocks(a, i * nbk + ks.astype(np.int64))
        bb = gc.tree_blocks(b, ks.astype(np.int64) * nbk + j)
        want = oracle.group_product(ab, bb, ks, depth)
        mine = gc.tree_blocks(c, [i * nbk + j])[0]
        assert np.array_equal(mine.view(np.uint8), want.view(np.uint8)), ("C block", i, j, len(ks))
    # C's whole pyramid from every retained block (zero products included)
    leaf_nsq = np.zeros(nbk * nbk)
    leaf_occ = np.zeros(nbk * nbk, np.uint8)
    for s in range(0, len(groups), 8192):
        ids = groups[s:s + 8192]
        nsq, occ = oracle.leaf_norms(gc.tree_blocks(c, ids))
        leaf_nsq[ids] = nsq
        leaf_occ[ids] = occ
    want_nsq, want_occ = oracle.pyramid_from_leaves(leaf_nsq, leaf_occ, depth)
    got_nsq, got_occ = _pyr(c)
    assert np.array_equal(got_occ, want_occ), "C occupancy pyramid"
    assert np.array_equal(got_nsq.view(np.uint64), want_nsq.view(np.uint64)), "C norm pyramid"
    return len(groups)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_c5_full_size_vs_oracle(dtype):
    """BASELINE config 5 at n = 65536 (inputs generated on the GPU: > 100 GB of
    host staging otherwise), A = B = sym(u * 0.98^|i-j|), leaf 64, tau = 1e-8."""
    import torch

    from paper_1011_3534_b200 import workloads

    tdt = torch.float32 if dtype == "f32" else torch.float64
    at, _, leaf, taus = workloads.make_config_device("c5", "cuda:0", tdt)
    n = at.shape[0]
    a = sp.from_device_pointer(at.data_ptr(), n, leaf_size=leaf,
                               dtype=np.float32 if dtype == "f32" else np.float64)
    del at
    torch.cuda.empty_cache()
    c, st, det = sp.spamm_detailed(a, a, sp.SpammConfig(tau=taus[0], collect_boxes=True),
                                   keep_triples=True)
    assert 700_000 < st.leaf_matmuls < 850_000
    ngroups = check_product_vs_oracle(a, a, c, st, det, taus[0])
    assert ngroups == det.n_groups


def test_c4_first_sweeps_vs_oracle():
    """BASELINE config 4's first three SP2 sweeps at full size (32^3 Morton
    lattice, n = 32768, leaf 64, tau = 1e-7): every square X^2 checked against
    the oracle on the same iterate; the iterate then
    advances through the drop-in tc2_step (purification.py:105-134)."""
    import torch

    from paper_1011_3534_b200 import purification as P
    from paper_1011_3534_b200 import workloads

    L, leaf, tau = 32, 64, 1e-7
    n = L ** 3
    h = workloads.cubic_lattice_hamiltonian_device(L, "cuda:0")
    f = sp.from_device_pointer(h.data_ptr(), n, leaf_size=leaf)
    del h
    torch.cuda.empty_cache()
    x = P.tc2_initial_guess(f)
    retained = []
    for sweep in range(3):
        c, st, det = sp.spamm_detailed(x, x, sp.SpammConfig(tau=tau, collect_boxes=True),
                                       keep_triples=True)
        check_product_vs_oracle(x, x, c, st, det, tau, n_sample=16, seed=sweep)
        retained.append(st.leaf_matmuls)
        del c
        x, _ = P.tc2_step(x, n // 2, P.SpammMode(tau))
    assert retained[0] > 0 and retained[2] >= retained[0]
