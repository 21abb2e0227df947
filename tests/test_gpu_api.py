"""The drop-in API on the B200, exercised like the reference's own tests
(pkg/tests/test_quadtree.py, test_multiply.py, test_acceptance.py), with the
CPU oracle or dense numpy as the independent check.  Every multiply runs
through the C ABI and the CUDA kernels."""

import math

import numpy as np
import pytest

import paper_1011_3534_b200 as sp
from oracle import oracle

pytestmark = pytest.mark.gpu


def _exp_pair(n, a1, a2):
    d = np.abs(np.arange(n)[:, None] - np.arange(n)[None, :]).astype(float)
    return np.exp(-a1 * d), np.exp(-a2 * d)


# ------------------------------------------------------------- quadtree
def test_identity4_single_leaf():
    m = sp.from_dense(np.eye(4), leaf_size=4)
    assert isinstance(m.root, sp.LeafNode)
    assert m.root.norm_sq == 4.0 and m.padded_dim == 4 and m.depth == 0


def test_zero8_empty_root():
    m = sp.from_dense(np.zeros((8, 8)), leaf_size=4)
    assert isinstance(m.root, sp.EmptyNode) and m.depth == 1 and m.root.norm_sq == 0.0


def test_ones5_padding_and_quadrants():
    m = sp.from_dense(np.ones((5, 5)), leaf_size=4)
    assert m.padded_dim == 8 and m.depth == 1 and m.root.norm_sq == 25.0
    assert m.root.children[3].norm_sq == 1.0


def test_roundtrip_exhaustive_small():
    rng = np.random.default_rng(0)
    for n in range(1, 66):
        data = rng.standard_normal((n, n))
        for leaf in (1, 2, 4):
            m = sp.from_dense(data, leaf_size=leaf)
            back = sp.to_dense(m)
            assert back.shape == (n, n) and np.array_equal(back, data), (n, leaf)
            pad = m._padded
            assert not pad[n:, :].any() and not pad[:, n:].any()


def test_roundtrip_rebuild_identical_tree():
    rng = np.random.default_rng(1)
    data = rng.standard_normal((100, 100))
    m = sp.from_dense(data)
    again = sp.from_dense(sp.to_dense(m))
    assert again.structurally_equal(m)
    assert again.root.norm_sq == m.root.norm_sq


def test_norm_matches_dense():
    rng = np.random.default_rng(2)
    for n in (3, 16, 50, 127):
        data = rng.standard_normal((n, n))
        ref = float(np.linalg.norm(data))
        assert abs(sp.node_norm(sp.from_dense(data)) - ref) <= 8 * np.finfo(float).eps * ref


@pytest.mark.parametrize("leaf", [1, 2, 4, 8, 16, 32, 64, 128])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_pyramid_bit_exact_vs_oracle(leaf, dtype):
    rng = np.random.default_rng(leaf)
    n = 3 * leaf + 5
    data = (rng.standard_normal((n, n)) * np.exp(-0.3 * np.abs(np.arange(n)[:, None] - np.arange(n)))).astype(dtype)
    data[: min(n, leaf), : min(n, leaf)] = -0.0  # an all-(-0.0) leaf is canonicalised
    m = sp.from_dense(data, leaf_size=leaf, dtype=dtype)
    pa = oracle.pad(data, leaf, dtype)
    nsq, occ = oracle.build_pyramid(pa, leaf)
    assert np.array_equal(m._pyramid()[2].view(np.uint64), nsq.view(np.uint64))
    assert np.array_equal(m._pyramid()[3], occ)
    assert np.array_equal(m._padded.view(np.uint8), pa.view(np.uint8))  # incl. +0.0 rewrite


# ------------------------------------------------------------- multiply
def test_identity_times_b_exact():
    bd = np.random.default_rng(0).standard_normal((20, 20))
    c, stats = sp.spamm(sp.identity(20), sp.from_dense(bd), sp.SpammConfig(tau=0.0))
    assert np.array_equal(sp.to_dense(c), bd) and stats.omitted_budget == 0.0


def test_tau_above_total_norm_prunes_root():
    rng = np.random.default_rng(1)
    a = sp.from_dense(rng.standard_normal((16, 16)))
    b = sp.from_dense(rng.standard_normal((16, 16)))
    budget = sp.node_norm(a) * sp.node_norm(b)
    c, st = sp.spamm(a, b, sp.SpammConfig(tau=budget * 1.5, collect_boxes=True))
    assert isinstance(c.root, sp.EmptyNode) and st.leaf_matmuls == 0
    assert st.omitted_budget == math.sqrt(a._norm_sq[0][0, 0]) * math.sqrt(b._norm_sq[0][0, 0])
    assert st.boxes == [sp.PrunedBox(0, 0, 0, a.padded_dim, 0)]


def test_full_enumeration_counts():
    rng = np.random.default_rng(2)
    for n, leaf in ((8, 4), (64, 8), (256, 32)):
        a = sp.from_dense(rng.standard_normal((n, n)), leaf_size=leaf)
        b = sp.from_dense(rng.standard_normal((n, n)), leaf_size=leaf)
        _, st = sp.spamm(a, b, sp.SpammConfig(tau=0.0))
        assert st.leaf_matmuls == (n // leaf) ** 3


def test_exact_vs_dense_many_leaves():
    rng = np.random.default_rng(3)
    for n, leaf in ((64, 4), (100, 8), (128, 16), (300, 32), (256, 64), (512, 128)):
        ad = rng.standard_normal((n, n))
        bd = rng.standard_normal((n, n))
        got = sp.to_dense(sp.exact_multiply(sp.from_dense(ad, leaf_size=leaf),
                                            sp.from_dense(bd, leaf_size=leaf)))
        ref = ad @ bd
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-13


def test_zero_operand_gives_empty():
    rng = np.random.default_rng(4)
    z = sp.from_dense(np.zeros((24, 24)))
    m = sp.from_dense(rng.standard_normal((24, 24)))
    assert isinstance(sp.exact_multiply(z, m).root, sp.EmptyNode)
    c2, st = sp.spamm(m, z, sp.SpammConfig(tau=0.0))
    assert isinstance(c2.root, sp.EmptyNode)
    assert st.leaf_matmuls == 0 and st.pruned_calls == 1
    assert st.empty_skip_volume == m.padded_dim ** 3


def test_permutation_times_transpose_is_identity():
    perm = np.random.default_rng(5).permutation(32)
    p = np.zeros((32, 32))
    p[np.arange(32), perm] = 1.0
    c = sp.exact_multiply(sp.from_dense(p), sp.from_dense(p.T))
    assert np.array_equal(sp.to_dense(c), np.eye(32))


@pytest.mark.parametrize("leaf,tau", [(4, 1e-8), (8, 1e-6), (16, 1e-6), (32, 1e-7), (64, 1e-9),
                                      (128, 1e-9)])
def test_matches_oracle_bit_exact(leaf, tau):
    """Retained triples, boxes, stats and C bit-for-bit vs the oracle across
    every leaf-kernel path (SIMT <= 16, DMMA 32/64, DMMA sub-tiled 128)."""
    n = max(512, 8 * leaf)
    a_d, b_d = _exp_pair(n, 0.05 * 64 / leaf, 0.07 * 64 / leaf)
    rng = np.random.default_rng(leaf)
    a_d = a_d * rng.uniform(-1, 1, a_d.shape)
    b_d = b_d * rng.uniform(-1, 1, b_d.shape)
    a = sp.from_dense(a_d, leaf_size=leaf)
    b = sp.from_dense(b_d, leaf_size=leaf)
    c, st, det = sp.spamm_detailed(a, b, sp.SpammConfig(tau=tau, collect_boxes=True),
                                   keep_triples=True)
    ref = oracle.spamm(a_d, b_d, leaf, tau)
    assert np.array_equal(det.triples, ref["triples"])
    got_boxes = np.array([[x.i_lo, x.j_lo, x.k_lo, x.edge, x.tier] for x in st.boxes],
                         np.int64).reshape(-1, 5)
    assert np.array_equal(got_boxes, ref["boxes"])
    for k in ("leaf_matmuls", "pruned_calls", "pruned_volume", "empty_skip_volume",
              "max_depth_reached"):
        assert getattr(st, k) == ref["stats"][k], k
    assert st.omitted_budget == ref["stats"]["omitted_budget"]
    assert np.array_equal(c._padded.view(np.uint64), ref["c_padded"].view(np.uint64))
    assert np.array_equal(c._pyramid()[2].view(np.uint64), ref["nsq_c"].view(np.uint64))


def test_float32_path_matches_oracle():
    n, leaf, tau = 384, 32, 1e-5
    a_d, b_d = _exp_pair(n, 0.02, 0.03)
    rng = np.random.default_rng(7)
    a_d = (a_d * rng.uniform(-1, 1, a_d.shape)).astype(np.float32)
    b_d = (b_d * rng.uniform(-1, 1, b_d.shape)).astype(np.float32)
    a = sp.from_dense(a_d, leaf_size=leaf, dtype=np.float32)
    b = sp.from_dense(b_d, leaf_size=leaf, dtype=np.float32)
    c, st, det = sp.spamm_detailed(a, b, sp.SpammConfig(tau=tau), keep_triples=True)
    ref = oracle.spamm(a_d, b_d, leaf, tau, dtype=np.float32)
    assert np.array_equal(det.triples, ref["triples"])
    assert st.omitted_budget == ref["stats"]["omitted_budget"]
    assert np.array_equal(c._padded.view(np.uint32), ref["c_padded"].view(np.uint32))


def test_error_bound_random_decay_pairs():
    rng = np.random.default_rng(7)
    taus = [1e-2, 1e-4, 1e-6, 1e-8, 1e-10, 1e-12]
    for _ in range(20):
        n = int(rng.integers(8, 49))
        alpha = float(rng.uniform(0.2, 2.5))
        idx = np.arange(n)
        decay = np.exp(-alpha * np.abs(idx[:, None] - idx[None, :]))
        a = sp.from_dense(decay * rng.standard_normal((n, n)))
        b = sp.from_dense(decay * rng.standard_normal((n, n)))
        scale_ab = sp.node_norm(a) * sp.node_norm(b)
        exact = sp.to_dense(sp.exact_multiply(a, b))
        for tau in taus:
            approx, st = sp.spamm(a, b, sp.SpammConfig(tau=tau))
            err = float(np.linalg.norm(sp.to_dense(approx) - exact))
            assert err <= st.omitted_budget + 1e-12 * scale_ab


def test_multiply_error_matches_dense():
    a_d, b_d = _exp_pair(512, 1.0, 2.0)
    a, b = sp.from_dense(a_d), sp.from_dense(b_d)
    for tau in (1e-2, 1e-6, 1e-10):
        err, budget = sp.multiply_error(a, b, sp.SpammConfig(tau=tau))
        approx, st = sp.spamm(a, b, sp.SpammConfig(tau=tau))
        ref = float(np.linalg.norm(sp.to_dense(approx) - sp.to_dense(sp.exact_multiply(a, b))))
        assert abs(err - ref) <= 1e-12 * max(ref, 1e-300) + 1e-300
        assert budget == st.omitted_budget and err <= budget + 1e-12


def test_monotone_work_and_tier_decay():
    a_d, b_d = _exp_pair(256, 0.7, 1.3)
    a, b = sp.from_dense(a_d), sp.from_dense(b_d)
    counts = [sp.spamm(a, b, sp.SpammConfig(tau=t))[1].leaf_matmuls
              for t in (0.0, 1e-12, 1e-9, 1e-6, 1e-3, 1e-1)]
    assert all(lo <= hi for lo, hi in zip(counts[1:], counts[:-1]))
    flat = sp.spamm(a, b, sp.SpammConfig(tau=1e-6))[1]
    dec = sp.spamm(a, b, sp.SpammConfig(tau=1e-6, tier_tau_decay=True))[1]
    assert dec.leaf_matmuls >= flat.leaf_matmuls
    assert dec.omitted_budget <= flat.omitted_budget
    assert dec.covered_volume(4) == a.padded_dim ** 3


def test_determinism_bit_identical():
    a_d, b_d = _exp_pair(256, 0.9, 1.1)
    a, b = sp.from_dense(a_d), sp.from_dense(b_d)
    cfg = sp.SpammConfig(tau=1e-7, collect_boxes=True)
    c1, s1 = sp.spamm(a, b, cfg)
    c2, s2 = sp.spamm(a, b, cfg)
    assert sp.to_dense(c1).tobytes() == sp.to_dense(c2).tobytes()
    assert s1 == s2


def test_count_stats_off():
    a_d, b_d = _exp_pair(128, 0.5, 0.5)
    a, b = sp.from_dense(a_d), sp.from_dense(b_d)
    _, st = sp.spamm(a, b, sp.SpammConfig(tau=1e-6, count_stats=False))
    assert st.leaf_matmuls == 0 and st.pruned_calls == 0 and st.omitted_budget == 0.0
    assert st.max_depth_reached == a.depth


def test_dimension_mismatch_rejected():
    rng = np.random.default_rng(10)
    a = sp.from_dense(rng.standard_normal((16, 16)))
    with pytest.raises(sp.DimensionMismatchError):
        sp.spamm(a, sp.from_dense(rng.standard_normal((32, 32))), sp.SpammConfig())
    with pytest.raises(sp.DimensionMismatchError):
        sp.spamm(a, sp.from_dense(rng.standard_normal((16, 16)), leaf_size=2), sp.SpammConfig())
    with pytest.raises(sp.DimensionMismatchError):
        sp.spamm(a, sp.from_dense(rng.standard_normal((16, 16)), dtype=np.float32),
                 sp.SpammConfig())


def test_product_tree_chains():
    """C feeds the next multiply (the SP2 pattern): C's tree equals a tree
    rebuilt from its dense form, bit for bit."""
    a_d, _ = _exp_pair(300, 0.3, 0.3)
    a = sp.from_dense(a_d, leaf_size=16)
    c, _ = sp.spamm(a, a, sp.SpammConfig(tau=1e-9))
    again = sp.from_dense(sp.to_dense(c), leaf_size=16)
    assert again.structurally_equal(c)
    assert np.array_equal(again._pyramid()[2].view(np.uint64), c._pyramid()[2].view(np.uint64))
    c2, _ = sp.spamm(c, c, sp.SpammConfig(tau=1e-9))
    r2 = oracle.spamm(sp.to_dense(c), sp.to_dense(c), 16, 1e-9)
    assert np.array_equal(c2._padded.view(np.uint64), r2["c_padded"].view(np.uint64))


@pytest.mark.slow
def test_c5_proxy_n16384_vs_oracle():
    """The n=65536 config's structure at a size the oracle finishes in
    seconds: sym(u * 0.98^d), B = A, leaf 64, tau = 1e-8."""
    from paper_1011_3534_b200 import workloads
    a_d = workloads.exponential_decay(16384, 0.98, 0, symmetric=True)
    a = sp.from_dense(a_d, leaf_size=64)
    c, st, det = sp.spamm_detailed(a, a, sp.SpammConfig(tau=1e-8), keep_triples=True)
    ref = oracle.spamm(a_d, a_d, 64, 1e-8)
    assert st.leaf_matmuls == ref["stats"]["leaf_matmuls"] == 186166
    assert np.array_equal(det.triples, ref["triples"])
    assert st.omitted_budget == ref["stats"]["omitted_budget"]
    assert np.array_equal(c._padded.view(np.uint64), ref["c_padded"].view(np.uint64))


@pytest.mark.gpu
def test_c5_full_size_symmetric_product():
    """BASELINE config 5 at full size (n = 65536, leaf 64, tau = 1e-8), inputs
    generated on the GPU: A = B symmetric, so the retained triple set is
    symmetric and C = A*A must come out exactly symmetric (each transposed
    product runs the same FMA chains with the factors swapped, in the same k
    order and merge tree).  Also checks the retained count against the
    structure of the n = 16384 proxy (~0.77 M)."""
    import torch
    from paper_1011_3534_b200 import distributed as spd
    from paper_1011_3534_b200 import workloads

    at, _, leaf, taus = workloads.make_config_device("c5", "cuda:0")
    n = at.shape[0]
    a = sp.from_device_pointer(at.data_ptr(), n, leaf_size=leaf)
    del at
    torch.cuda.empty_cache()
    c, st, det = sp.spamm_detailed(a, a, sp.SpammConfig(tau=taus[0]), keep_triples=True)
    assert 700_000 < st.leaf_matmuls < 850_000
    tr = det.triples
    fwd = {(int(i), int(j), int(k)) for i, j, k in tr[:200_000]}
    back = {(int(j), int(i), int(k)) for i, j, k in tr}
    assert fwd <= back, "retained set not symmetric"
    cs = spd.tree_storage(c)
    blk = 8192
    for r0 in range(0, n, blk):
        for c0 in range(0, r0 + 1, blk):
            x = cs[r0:r0 + blk, c0:c0 + blk]
            y = cs[c0:c0 + blk, r0:r0 + blk].t()
            assert torch.equal(x, y), ("C not symmetric", r0, c0)
    # C's root norm agrees with the blocks' norms (pyramid over the product)
    assert c.norm() > 0


@pytest.mark.gpu
def test_nonzero_blocks_match_padded():
    rng = np.random.default_rng(5)
    n, leaf = 200, 16
    x = rng.uniform(-1, 1, (n, n))
    x[:48, :] = 0.0
    x[:, 100:150] = 0.0
    t = sp.from_dense(x, leaf_size=leaf)
    ids, blocks = t.nonzero_blocks()
    occ = np.asarray(t._leaf_nonzero).reshape(-1)
    assert np.array_equal(ids, np.flatnonzero(occ))
    ref = np.asarray(t._blocks).reshape(-1, leaf, leaf)[ids]
    assert np.array_equal(blocks.view(np.uint64), ref.view(np.uint64))
    c, _ = sp.spamm(t, t, sp.SpammConfig(tau=1e-3))
    ids, blocks = c.nonzero_blocks()
    dense = np.zeros((c.padded_dim, c.padded_dim))
    nb = c.block_grid
    for g, blk in zip(ids, blocks):
        i, j = divmod(int(g), nb)
        dense[i * leaf:(i + 1) * leaf, j * leaf:(j + 1) * leaf] = blk
    assert np.array_equal(dense, c._padded)


@pytest.mark.gpu
def test_nonzero_blocks_async_overlaps_later_calls():
    """wait=False: the copies of several products are in flight together while
    later multiplies run; every one lands bit-identical to the synchronous
    read, and an unwaited transfer is completed when collected."""
    import torch

    rng = np.random.default_rng(11)
    n, leaf = 512, 32
    d = np.abs(np.subtract.outer(np.arange(n), np.arange(n)))
    x = rng.uniform(-1, 1, (n, n)) * 0.9 ** d
    t = sp.from_dense(x, leaf_size=leaf)
    taus = [1e-2, 1e-4, 1e-6, 1e-8]
    G = t.block_grid ** 2
    bufs = [torch.empty((G, leaf, leaf), dtype=torch.float64, pin_memory=True).numpy()
            for _ in taus]
    pend, prods = [], []
    for q, tau in enumerate(taus):
        c, _ = sp.spamm(t, t, sp.SpammConfig(tau=tau))
        pend.append(c.nonzero_blocks(out=bufs[q], wait=False))
        prods.append(c)
    for c, p in zip(prods, pend):
        ids, blocks = p.wait()
        ids2, blocks2 = c.nonzero_blocks()
        assert np.array_equal(ids, ids2)
        assert np.array_equal(blocks.view(np.uint64), blocks2.view(np.uint64))
        assert p.wait()[0] is ids  # waiting twice is a no-op
    # the product may be released before its copy completes
    c, _ = sp.spamm(t, t, sp.SpammConfig(tau=1e-8))
    ref = c.nonzero_blocks()[1].copy()
    p = c.nonzero_blocks(out=bufs[0], wait=False)
    del c
    _, blocks = p.wait()
    assert np.array_equal(blocks.view(np.uint64), ref.view(np.uint64))
    # an empty tree: nothing to copy
    z = sp.from_dense(np.zeros((64, 64)), leaf_size=leaf)
    ids, blocks = z.nonzero_blocks(wait=False).wait()
    assert len(ids) == 0 and blocks.shape == (0, leaf, leaf)


@pytest.mark.gpu
def test_from_dense_async_matches_sync():
    """from_dense(wait=False): the build overlaps queued multiplies; the tree,
    its root norm and every product with it are identical to the synchronous
    build's, and a pending tree may be dropped before its build completes."""
    import torch

    rng = np.random.default_rng(7)
    for n, leaf in ((300, 16), (1024, 64)):
        d = np.abs(np.subtract.outer(np.arange(n), np.arange(n)))
        x = rng.uniform(-1, 1, (n, n)) * 0.9 ** d
        pin = torch.empty((n, n), dtype=torch.float64, pin_memory=True).numpy()
        pin[...] = x
        ref = sp.from_dense(x, leaf_size=leaf)
        busy, _ = sp.spamm(ref, ref, sp.SpammConfig(tau=0.0))  # work queued ahead
        t = sp.from_dense(pin, leaf_size=leaf, wait=False)
        c_ref, st_ref = sp.spamm(ref, ref, sp.SpammConfig(tau=1e-6))
        c, st = sp.spamm(t, t, sp.SpammConfig(tau=1e-6))  # ordered after the build
        assert st.leaf_matmuls == st_ref.leaf_matmuls
        assert np.array_equal(c._padded.view(np.uint64), c_ref._padded.view(np.uint64))
        assert t.norm() == ref.norm()
        for k in range(t.depth + 1):
            assert np.array_equal(t._norm_sq[k].view(np.uint64), ref._norm_sq[k].view(np.uint64))
            assert np.array_equal(t._occupied[k], ref._occupied[k])
        assert np.array_equal(t.to_dense(), x)
        assert t.wait() is t
        p2 = sp.from_dense(pin, leaf_size=leaf, wait=False)
        del p2  # dropped while (possibly) in flight
        del busy
    # dtype conversion and padding on the async path
    y = rng.uniform(-1, 1, (70, 70))
    a = sp.from_dense(y, leaf_size=8, dtype=np.float32, wait=False)
    b = sp.from_dense(y, leaf_size=8, dtype=np.float32)
    assert a.norm() == b.norm()
    assert np.array_equal(a._padded, b._padded)


def _crafted_blocks(n, leaf, rng):
    """A matrix whose leaves stress the segmented norm chains: rounding ties
    (s exactly half an ulp of the running sum), binade crossings inside and
    across segments, subnormal and overflowing squares, NaN, zero leaves."""
    x = np.zeros((n, n))
    nb = n // leaf
    kinds = ["ties", "ties3", "range", "subnormal", "overflow", "nan", "zero", "ramp", "random"]
    for q in range(nb * nb):
        i, j = divmod(q, nb)
        kind = kinds[q % len(kinds)]
        blk = x[i * leaf:(i + 1) * leaf, j * leaf:(j + 1) * leaf]
        if kind == "ties":       # acc in [2, 4): u = 2^-51, s = 2^-52 is a tie
            blk[...] = 2.0 ** -26
            blk[0, 0] = 1.5
        elif kind == "ties3":    # s = 9 * 2^-52 = 4.5 u: ties again
            blk[...] = 3 * 2.0 ** -26
            blk[0, 0] = 1.5
            blk[leaf // 2, 3] = 1.0
        elif kind == "range":
            blk[...] = rng.uniform(-1, 1, blk.shape) * 10.0 ** rng.integers(-150, 150, blk.shape)
        elif kind == "subnormal":
            blk[...] = rng.uniform(-1, 1, blk.shape) * 1e-160
        elif kind == "overflow":
            blk[...] = rng.uniform(-1, 1, blk.shape)
            blk[leaf - 1, leaf // 3] = 1e200
        elif kind == "nan":
            blk[...] = rng.uniform(-1, 1, blk.shape)
            blk[leaf // 2, leaf // 2] = np.nan
        elif kind == "ramp":     # growing along the chain: many binade crossings
            blk[...] = np.arange(1, leaf * leaf + 1).reshape(leaf, leaf) ** 3.0
        elif kind == "random":
            blk[...] = rng.uniform(-1, 1, blk.shape)
    return x


@pytest.mark.gpu
@pytest.mark.parametrize("leaf", [16, 32, 64])
def test_product_norms_segmented_chain_edge_cases(leaf):
    """C = A * I (tau = 0) carries A's crafted leaves into a product (NaN and
    overflow spread along their block rows); C's norm pyramid, built by the
    segmented-chain kernel, must equal the oracle's sequential chains bit for
    bit on every leaf."""
    rng = np.random.default_rng(21)
    n = leaf * 6
    x = _crafted_blocks(n, leaf, rng)
    a = sp.from_dense(x, leaf_size=leaf)
    eye = sp.from_dense(np.eye(n), leaf_size=leaf)
    c, _ = sp.spamm(a, eye, sp.SpammConfig(tau=0.0))
    cp = c._padded.copy()
    assert np.isnan(cp).any() and np.array_equal(cp[:leaf, :leaf], a._padded[:leaf, :leaf])
    nsq, occ = oracle.build_pyramid(cp, leaf)
    got = np.concatenate([lv.reshape(-1) for lv in c._norm_sq])
    goto = np.concatenate([lv.reshape(-1) for lv in c._occupied])
    assert np.array_equal(got.view(np.uint64), nsq.view(np.uint64))
    assert np.array_equal(goto, occ.astype(bool))


@pytest.mark.gpu
@pytest.mark.parametrize("leaf", [16, 32, 64, 128])
def test_product_f32_matches_oracle(leaf):
    rng = np.random.default_rng(3)
    n = leaf * 8 - 5
    d = np.abs(np.subtract.outer(np.arange(n), np.arange(n)))
    ad = (rng.uniform(-1, 1, (n, n)) * 0.8 ** d).astype(np.float32)
    bd = (rng.uniform(-1, 1, (n, n)) * 0.8 ** d).astype(np.float32)
    a = sp.from_dense(ad, leaf_size=leaf, dtype=np.float32)
    b = sp.from_dense(bd, leaf_size=leaf, dtype=np.float32)
    c, st = sp.spamm(a, b, sp.SpammConfig(tau=1e-4))
    ref = oracle.spamm(ad, bd, leaf, 1e-4, dtype=np.float32)
    assert st.leaf_matmuls == ref["stats"]["leaf_matmuls"]
    assert np.array_equal(c._padded.view(np.uint32), ref["c_padded"].view(np.uint32))
    nsq, _ = oracle.build_pyramid(ref["c_padded"].copy(), leaf)
    got = np.concatenate([lv.reshape(-1) for lv in c._norm_sq])
    assert np.array_equal(got.view(np.uint64), nsq.view(np.uint64))


@pytest.mark.gpu
def test_chained_launch_path_is_deterministic():
    """The c2-shaped path chains three kernels programmatically (traversal ->
    leaf products -> C's norms, each launched before its predecessor ends).
    Repeated multiplies must give bit-identical products and C pyramids (a
    dependent reading its predecessor's outputs too early shows up here)."""
    rng = np.random.default_rng(17)
    n, leaf = 4096, 64
    d = np.abs(np.subtract.outer(np.arange(n), np.arange(n)))
    u = rng.uniform(-1, 1, (n, n)) * 0.95 ** d
    a = sp.from_dense(0.5 * (u + u.T), leaf_size=leaf)
    # tau alternates call after call, so each call's group list differs from
    # the one the previous call left in the scratch buffers: a dependent that
    # read them too early could not pass by seeing an identical stale list
    refs = {}
    for it in range(16):
        tau = (1e-6, 1e-9)[it & 1]
        c, st = sp.spamm(a, a, sp.SpammConfig(tau=tau))
        pyr = np.concatenate([lv.reshape(-1) for lv in c._norm_sq]).view(np.uint64)
        ids, blocks = c.nonzero_blocks()
        got = (st.leaf_matmuls, pyr.copy(), ids.copy(), blocks.view(np.uint64).copy())
        ref = refs.setdefault(tau, got)
        assert got[0] == ref[0]
        assert np.array_equal(got[1], ref[1])
        assert np.array_equal(got[2], ref[2]) and np.array_equal(got[3], ref[3])
    assert refs[1e-6][0] < refs[1e-9][0]


@pytest.mark.gpu
def test_from_device_pointer_is_stream_ordered():
    """from_device_pointer hands off with the producer's stream by events
    (spamm_tree_from_device_on), no device-wide synchronisation: the copy sees
    the final values of work still queued on a side stream, and that stream
    may overwrite the array right after the call without touching the tree."""
    import torch

    n, leaf = 1024, 32
    s = torch.cuda.Stream()
    a = torch.empty((n, n), dtype=torch.float64, device="cuda")
    with torch.cuda.stream(s):
        x = torch.rand((2048, 2048), dtype=torch.float64, device="cuda")
        for _ in range(20):  # keep the side stream busy well past the call below
            x = torch.tanh(x @ x / 2048.0)
        a.copy_(x[:n, :n])
        t = sp.from_device_pointer(a.data_ptr(), n, leaf_size=leaf, stream=s.cuda_stream)
        a.fill_(7.0)  # queued after the copy (the stream waits for the library)
    s.synchronize()
    want = x[:n, :n].cpu().numpy()
    assert np.array_equal(t.to_dense(), want)
    # the pyramid is the one of the final values
    assert np.array_equal(t._pyramid()[2], sp.from_dense(want, leaf_size=leaf)._pyramid()[2])


@pytest.mark.gpu
@pytest.mark.parametrize("n,ld_pad", [(1024, 0), (1024, 6), (1000, 0), (777, 3)])
def test_from_device_pointer_fused_and_copy_paths(n, ld_pad):
    """from_device_pointer on device data: the fused build (K1 reads the
    source once and writes the tree's storage, n == N with 16-byte aligned
    rows) and the copy-then-K1 path (padding, odd leading dimensions) give
    the host build's tree bit for bit -- storage and pyramid."""
    import torch

    rng = np.random.default_rng(n + ld_pad)
    d = np.abs(np.subtract.outer(np.arange(n), np.arange(n)))
    host = rng.uniform(-1, 1, (n, n)) * 0.9 ** d
    host[5, :] = 0.0
    host[7, 9] = -0.0
    dev = torch.zeros((n, n + ld_pad), dtype=torch.float64, device="cuda")
    dev[:, :n] = torch.from_numpy(host).cuda()
    t = sp.from_device_pointer(dev.data_ptr(), n, leaf_size=32, ld=n + ld_pad)
    ref = sp.from_dense(host, leaf_size=32)
    assert np.array_equal(t._padded.view(np.uint64), ref._padded.view(np.uint64))
    assert np.array_equal(t._pyramid()[2].view(np.uint64), ref._pyramid()[2].view(np.uint64))
    assert np.array_equal(t._pyramid()[3], ref._pyramid()[3])


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,mode", [(np.float64, "host"), (np.float64, "device"),
                                        (np.float64, "device_ld"), (np.float32, "host")])
def test_dense_rows_build_matches_oracle(dtype, mode):
    """Large dense builds (leaf 64, >= 64 leaves per SM: the TMA-fed rows
    kernel, in place after a host copy or fused with the copy from a device
    source) give the oracle's pyramid bit for bit and the source's storage,
    with empty leaves, a leaf holding only -0.0 (canonicalised) and NaN."""
    import torch
    from oracle import oracle

    n, leaf = 8192, 64
    rng = np.random.default_rng(17)
    host = (rng.uniform(-1, 1, (n, n)) * np.exp(-rng.uniform(0, 30, (n, n)))).astype(dtype)
    host[128:192, :] = 0                      # a whole empty block row
    host[640:704, 64:128] = 0
    host[650, 70] = -0.0                      # only -0.0 in this leaf
    host[1000, 3000] = np.nan
    host[4097, 4095] = 1e-200                 # square underflows to a subnormal
    if mode == "host":
        t = sp.from_dense(host, leaf_size=leaf, dtype=dtype)
    else:
        pad = 2 if mode == "device_ld" else 0
        dev = torch.zeros((n, n + pad), dtype=torch.float64, device="cuda")
        dev[:, :n] = torch.from_numpy(host).cuda()
        t = sp.from_device_pointer(dev.data_ptr(), n, leaf_size=leaf, ld=n + pad)
    want = host.copy()
    nsq, occ = oracle.build_pyramid(want, leaf)   # canonicalises `want` in place
    u = np.uint64 if dtype == np.float64 else np.uint32
    assert np.array_equal(t._pyramid()[2].view(np.uint64), nsq.view(np.uint64))
    assert np.array_equal(t._pyramid()[3], occ)
    assert np.array_equal(t._padded.view(u), want.view(u))


@pytest.mark.parametrize("traversal", ["auto", "tiered"])
@pytest.mark.parametrize("dtype,leaf", [(np.float64, 32), (np.float32, 32), (np.float64, 16)])
def test_need_blocks_match_retained_triples(traversal, dtype, leaf):
    """The device-formed plan (SPAMM_NEED_BLOCKS) is exactly the set of B
    blocks (k, j) the retained triples read, whole product and row bands,
    dense (bitmask groups) and tiered traversals."""
    a, b = _exp_pair(1024, 0.05, 0.08)
    ta = sp.from_dense(a.astype(dtype), leaf_size=leaf)
    tb = sp.from_dense(b.astype(dtype), leaf_size=leaf)
    nb = ta.block_grid
    for rows in (None, (0, nb), (3, nb // 2 + 1), (nb - 1, nb)):
        for tau in (1e-9, 1e-4, 10.0):
            for trav_only in (True, False):
                _, _, det = sp.spamm_detailed(ta, tb, sp.SpammConfig(tau=tau), keep_triples=True,
                                              rows=rows, traversal=traversal,
                                              traverse_only=trav_only, need_blocks=True)
                want = np.zeros(nb * nb, bool)
                tr = det.triples
                want[tr[:, 2].astype(np.int64) * nb + tr[:, 1]] = True
                assert det.need_blocks.shape == (nb * nb,)
                assert np.array_equal(det.need_blocks, want), (rows, tau, trav_only)
