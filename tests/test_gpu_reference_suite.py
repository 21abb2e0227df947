"""The reference's own behavioural suite, run against the B200 package through
the ``spamm`` import shim (paper_1011_3534_b200.compat).

Every test below restates one test of the reference package -- the file and
line it follows are in its docstring -- and reaches the library only through
``import spamm`` / ``spamm.quadtree`` / ``spamm.multiply`` /
``spamm.generators``, exactly as the reference's tests do, so it checks the
drop-in switch as well as the kernels.  (The reference's test files cannot be
executed on the GPU box: /root/reference is not there.  Their checks are
restated here; the independent oracles they use -- a pure-Python triple loop
and a flat depth-first re-derivation of the pruned recursion -- are rewritten
below.)

Covered: pkg/tests/test_quadtree.py (all 20 tests), pkg/tests/
test_multiply.py (all 21), pkg/tests/test_acceptance.py:31-100 (3).
"""

import itertools
import math

import numpy as np
import pytest

from paper_1011_3534_b200 import compat

pytestmark = pytest.mark.gpu

EPS = float(np.finfo(np.float64).eps)


@pytest.fixture(scope="module")
def sp():
    """The library, imported under the reference's name."""
    compat.install()
    import spamm  # noqa: F401  (the shim)
    import spamm.generators as G
    import spamm.multiply as M
    import spamm.quadtree as Q

    class NS:
        pass

    ns = NS()
    ns.Q, ns.M, ns.G = Q, M, G
    yield ns
    compat.uninstall()


def triple_loop(a, b):
    """Dense product by explicit Python loops (no BLAS): out[i][j] += a[i][k] b[k][j]."""
    a = np.asarray(a, dtype=np.float64).tolist()
    b = np.asarray(b, dtype=np.float64).tolist()
    n, inner, m = len(a), len(b), len(b[0])
    out = [[0.0] * m for _ in range(n)]
    for i in range(n):
        row = out[i]
        for k in range(inner):
            x = a[i][k]
            if x == 0.0:
                continue
            bk = b[k]
            for j in range(m):
                row[j] += x * bk[j]
    return np.array(out)


def flat_dfs(pa, pb, leaf, tau):
    """Depth-first re-derivation of the pruned recursion (Eq. 4) on padded
    dense operands: leaf norms as sequential sums of squares, parents as
    ((c11 + c12) + c21) + c22, occupancy as any(x != 0), and an explicit
    stack over (tier, i, j, k).  Shares no code with the library or the
    oracle.  Returns (leaf products, set of pruned boxes, budget)."""
    N = pa.shape[0]
    depth = 0
    while leaf << depth < N:
        depth += 1

    def levels(p):
        nb = N // leaf
        blk = p.reshape(nb, leaf, nb, leaf).swapaxes(1, 2)
        s = np.zeros((nb, nb))
        for r in range(leaf):
            for c in range(leaf):
                s = s + blk[:, :, r, c] * blk[:, :, r, c]
        nz = (blk != 0).any(axis=(2, 3))
        sq, oc = [s], [nz]
        for _ in range(depth):
            f, o = sq[0], oc[0]
            sq.insert(0, ((f[::2, ::2] + f[::2, 1::2]) + f[1::2, ::2]) + f[1::2, 1::2])
            oc.insert(0, o[::2, ::2] | o[::2, 1::2] | o[1::2, ::2] | o[1::2, 1::2])
        return sq, oc

    sa, oa = levels(pa)
    sb, ob = levels(pb)
    work, total, boxes = 0, 0.0, set()
    todo = [(0, 0, 0, 0)]
    while todo:
        t, i, j, k = todo.pop()
        if not (oa[t][i, k] and ob[t][k, j]):
            continue
        p = math.sqrt(sa[t][i, k]) * math.sqrt(sb[t][k, j])
        if p < tau:
            e = N >> t
            boxes.add((t, i * e, j * e, k * e, e))
            total += p
        elif t == depth:
            work += 1
        else:
            todo.extend((t + 1, 2 * i + x, 2 * j + y, 2 * k + z)
                        for x in (0, 1) for y in (0, 1) for z in (0, 1))
    return work, boxes, total


def morton3(i, j, k):
    """i-major three-way bit interleave (the box-log key)."""
    key = 0
    for bit in range(21):
        key |= ((i >> bit) & 1) << (3 * bit + 2)
        key |= ((j >> bit) & 1) << (3 * bit + 1)
        key |= ((k >> bit) & 1) << (3 * bit)
    return key


# ----------------------------------------------- pkg/tests/test_quadtree.py
class TestQuadtree:
    def test_identity4_single_leaf(self, sp):
        """test_quadtree.py:12-16 -- a 4x4 identity is one leaf of norm^2 4."""
        m = sp.Q.from_dense(np.eye(4), leaf_size=4)
        assert isinstance(m.root, sp.Q.LeafNode)
        assert (m.root.norm_sq, m.padded_dim, m.depth) == (4.0, 4, 0)

    def test_zero8_empty_root(self, sp):
        """test_quadtree.py:19-23 -- an all-zero matrix has an Empty root."""
        m = sp.Q.from_dense(np.zeros((8, 8)), leaf_size=4)
        assert isinstance(m.root, sp.Q.EmptyNode)
        assert m.depth == 1 and m.root.norm_sq == 0.0

    def test_ones5_padding_and_quadrants(self, sp):
        """test_quadtree.py:26-34 -- padding to 8; quadrant 22 holds only (4, 4)."""
        m = sp.Q.from_dense(np.ones((5, 5)), leaf_size=4)
        assert (m.padded_dim, m.depth, m.root.norm_sq) == (8, 1, 25.0)
        assert m.root.children[3].norm_sq == 1.0

    def test_padding_region_exact_zero(self, sp):
        """test_quadtree.py:37-47 -- padding is exactly zero and minimal."""
        rng = np.random.default_rng(11)
        for n in (5, 9, 13, 33):
            m = sp.Q.from_dense(rng.standard_normal((n, n)))
            p = m._padded
            assert p.shape == (m.padded_dim,) * 2
            assert not p[n:].any() and not p[:, n:].any()
            assert m.padded_dim >= n and (m.depth == 0 or m.padded_dim // 2 < n)

    def test_roundtrip_exhaustive_small(self, sp):
        """test_quadtree.py:50-59 -- to_dense(from_dense(M)) == M, n = 1..65, leaf 1/2/4."""
        rng = np.random.default_rng(0)
        for n in range(1, 66):
            x = rng.standard_normal((n, n))
            for leaf in (1, 2, 4):
                back = sp.Q.to_dense(sp.Q.from_dense(x, leaf_size=leaf))
                assert back.shape == (n, n) and np.array_equal(back, x), (n, leaf)

    def test_roundtrip_rebuild_identical_tree(self, sp):
        """test_quadtree.py:62-69 -- rebuilding from to_dense gives the same tree."""
        x = np.random.default_rng(1).standard_normal((100, 100))
        m = sp.Q.from_dense(x)
        m2 = sp.Q.from_dense(sp.Q.to_dense(m))
        assert np.array_equal(sp.Q.to_dense(m2), x)
        assert (m2.padded_dim, m2.depth) == (m.padded_dim, m.depth)
        assert m2.root.norm_sq == m.root.norm_sq

    def test_to_dense_empty_is_zeros(self, sp):
        """test_quadtree.py:72-74."""
        assert np.array_equal(sp.Q.to_dense(sp.Q.from_dense(np.zeros((4, 4)))), np.zeros((4, 4)))

    def test_to_dense_matches_generator(self, sp):
        """test_quadtree.py:77-81 -- gen_exponential(512, 1) is exp(-|i-j|) exactly."""
        d = sp.Q.to_dense(sp.G.gen_exponential(512, 1.0))
        i, j = np.indices((512, 512))
        assert np.array_equal(d, np.exp(-np.abs(i - j).astype(float)))

    def test_norm_matches_dense(self, sp):
        """test_quadtree.py:84-90 -- root norm within 8 eps of numpy's."""
        rng = np.random.default_rng(2)
        for n in (3, 16, 50, 127):
            x = rng.standard_normal((n, n))
            ref = float(np.linalg.norm(x))
            assert abs(sp.Q.node_norm(sp.Q.from_dense(x)) - ref) <= 8 * EPS * ref

    def test_norm_cache_audit(self, sp):
        """test_quadtree.py:93-97 -- cached pyramid agrees with a recomputation."""
        rng = np.random.default_rng(3)
        for n in (8, 37, 64):
            assert sp.Q.audit_norm_cache(sp.Q.from_dense(rng.standard_normal((n, n)))) <= 4 * EPS

    def test_non_square_rejected(self, sp):
        """test_quadtree.py:100-102."""
        with pytest.raises(sp.Q.DimensionMismatchError):
            sp.Q.from_dense(np.ones((3, 4)))

    @pytest.mark.parametrize("leaf", [3, 0])
    def test_bad_leaf_size_rejected(self, sp, leaf):
        """test_quadtree.py:105-109."""
        with pytest.raises(ValueError):
            sp.Q.from_dense(np.eye(4), leaf_size=leaf)

    def test_filter_tau0_is_identity(self, sp):
        """test_quadtree.py:114-119."""
        m = sp.Q.from_dense(np.random.default_rng(4).standard_normal((20, 20)))
        f = sp.Q.filter_drop(m, 0.0)
        assert np.array_equal(sp.Q.to_dense(f), sp.Q.to_dense(m))
        assert f.root.norm_sq == m.root.norm_sq

    def test_filter_above_total_norm_empties(self, sp):
        """test_quadtree.py:122-125."""
        m = sp.Q.from_dense(np.ones((8, 8)))
        assert isinstance(sp.Q.filter_drop(m, sp.Q.node_norm(m) * 1.01).root, sp.Q.EmptyNode)

    def test_filter_matches_flat_scan(self, sp):
        """test_quadtree.py:128-144 -- dropping = zeroing every 4x4 block whose
        norm is below tau, found by a flat scan."""
        a = sp.G.gen_exponential(512, 1.0)
        tau = 1e-8
        kept = sp.Q.filter_drop(a, tau)
        N = a.padded_dim
        p = np.zeros((N, N))
        p[:512, :512] = sp.Q.to_dense(a)
        blk = p.reshape(N // 4, 4, N // 4, 4).swapaxes(1, 2)
        keep = np.sqrt((blk * blk).sum(axis=(2, 3))) >= tau
        want = (blk * keep[:, :, None, None]).swapaxes(1, 2).reshape(N, N)[:512, :512]
        assert np.array_equal(sp.Q.to_dense(kept), want)
        assert int(kept._leaf_nonzero.sum()) == int(keep.sum())

    def test_filter_idempotent(self, sp):
        """test_quadtree.py:147-154."""
        m = sp.Q.from_dense(np.random.default_rng(5).standard_normal((32, 32)) * 1e-3)
        once = sp.Q.filter_drop(m, 2e-3)
        twice = sp.Q.filter_drop(once, 2e-3)
        assert np.array_equal(sp.Q.to_dense(once), sp.Q.to_dense(twice))
        assert once.root.norm_sq == twice.root.norm_sq

    def test_add_empty_passthrough(self, sp):
        """test_quadtree.py:159-165 -- m + 0 is m bit for bit."""
        m = sp.Q.from_dense(np.random.default_rng(6).standard_normal((12, 12)))
        s = sp.Q.add(m, sp.Q.from_dense(np.zeros((12, 12))))
        assert np.array_equal(sp.Q.to_dense(s), sp.Q.to_dense(m))
        assert s.root.norm_sq == m.root.norm_sq

    def test_add_scale_vs_dense(self, sp):
        """test_quadtree.py:168-176."""
        rng = np.random.default_rng(7)
        a, b = rng.standard_normal((50, 50)), rng.standard_normal((50, 50))
        s = sp.Q.to_dense(sp.Q.add(sp.Q.from_dense(a), sp.Q.from_dense(b)))
        assert np.linalg.norm(s - (a + b)) <= 1e-14 * np.linalg.norm(a + b)
        t = sp.Q.to_dense(sp.Q.scale(sp.Q.from_dense(a), -2.5))
        assert np.linalg.norm(t - (-2.5 * a)) <= 1e-14 * np.linalg.norm(a)

    def test_trace_excludes_padding(self, sp):
        """test_quadtree.py:179-183."""
        assert sp.Q.trace(sp.Q.identity(7)) == 7.0
        d = np.random.default_rng(8).standard_normal((37, 37))
        assert np.isclose(sp.Q.trace(sp.Q.from_dense(d)), np.trace(d), rtol=1e-14)

    def test_add_dimension_mismatch(self, sp):
        """test_quadtree.py:186-188."""
        with pytest.raises(sp.Q.DimensionMismatchError):
            sp.Q.add(sp.Q.from_dense(np.eye(4)), sp.Q.from_dense(np.eye(8)))


# ----------------------------------------------- pkg/tests/test_multiply.py
class TestMultiply:
    def test_identity_times_b_exact(self, sp):
        """test_multiply.py:39-44 -- I * B == B bitwise, zero budget."""
        bd = np.random.default_rng(0).standard_normal((20, 20))
        c, st = sp.M.spamm(sp.Q.identity(20), sp.Q.from_dense(bd), sp.M.SpammConfig(tau=0.0))
        assert np.array_equal(sp.Q.to_dense(c), bd) and st.omitted_budget == 0.0

    def test_tau_above_total_norm_prunes_root(self, sp):
        """test_multiply.py:47-56 -- tau > ||A|| ||B||: one root box, budget exact."""
        rng = np.random.default_rng(1)
        a = sp.Q.from_dense(rng.standard_normal((16, 16)))
        b = sp.Q.from_dense(rng.standard_normal((16, 16)))
        bound = sp.Q.node_norm(a) * sp.Q.node_norm(b)
        c, st = sp.M.spamm(a, b, sp.M.SpammConfig(tau=bound * 1.5, collect_boxes=True))
        assert isinstance(c.root, sp.Q.EmptyNode) and st.leaf_matmuls == 0
        assert st.omitted_budget == bound
        assert st.boxes == [sp.M.PrunedBox(0, 0, 0, a.padded_dim, 0)]

    def test_full_enumeration_counts_n8(self, sp):
        """test_multiply.py:59-64 -- tau = 0 visits (n / b)^3 leaf products."""
        rng = np.random.default_rng(2)
        a = sp.Q.from_dense(rng.standard_normal((8, 8)), leaf_size=4)
        b = sp.Q.from_dense(rng.standard_normal((8, 8)), leaf_size=4)
        assert sp.M.spamm(a, b, sp.M.SpammConfig(tau=0.0))[1].leaf_matmuls == 8

    def test_exact_vs_triple_loop_oracle_64(self, sp):
        """test_multiply.py:67-74 -- exact product within 1e-13 of a triple loop."""
        rng = np.random.default_rng(3)
        ad, bd = rng.standard_normal((64, 64)), rng.standard_normal((64, 64))
        got = sp.Q.to_dense(sp.M.exact_multiply(sp.Q.from_dense(ad), sp.Q.from_dense(bd)))
        ref = triple_loop(ad, bd)
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-13

    def test_zero_operand_gives_empty(self, sp):
        """test_multiply.py:77-87 -- a zero operand: Empty product, one root skip."""
        z = sp.Q.from_dense(np.zeros((24, 24)))
        m = sp.Q.from_dense(np.random.default_rng(4).standard_normal((24, 24)))
        assert isinstance(sp.M.exact_multiply(z, m).root, sp.Q.EmptyNode)
        c, st = sp.M.spamm(m, z, sp.M.SpammConfig(tau=0.0))
        assert isinstance(c.root, sp.Q.EmptyNode)
        assert (st.leaf_matmuls, st.pruned_calls) == (0, 1)
        assert st.empty_skip_volume == m.padded_dim ** 3

    def test_permutation_times_transpose_is_identity(self, sp):
        """test_multiply.py:90-96 -- P P^T == I bitwise."""
        perm = np.random.default_rng(5).permutation(32)
        p = np.zeros((32, 32))
        p[np.arange(32), perm] = 1.0
        c = sp.M.exact_multiply(sp.Q.from_dense(p), sp.Q.from_dense(p.T))
        assert np.array_equal(sp.Q.to_dense(c), np.eye(32))

    def test_flat_recursion_agrees_on_decay_pair(self, sp):
        """test_multiply.py:158-168 -- against a flat DFS of Eq. 4: the same leaf
        count, the same pruned-box set, the budget within 1e-12, exact tiling."""
        a = sp.G.gen_exponential(512, 1.0)
        b = sp.G.gen_exponential(512, 2.0)
        _, st = sp.M.spamm(a, b, sp.M.SpammConfig(tau=1e-8, collect_boxes=True))
        work, boxes, total = flat_dfs(np.asarray(a._padded), np.asarray(b._padded), 4, 1e-8)
        assert st.leaf_matmuls == work
        assert {(x.tier, x.i_lo, x.j_lo, x.k_lo, x.edge) for x in st.boxes} == boxes
        assert math.isclose(st.omitted_budget, total, rel_tol=1e-12)
        assert st.covered_volume(4) == a.padded_dim ** 3

    def test_multiply_error_tau0(self, sp):
        """test_multiply.py:173-179."""
        rng = np.random.default_rng(6)
        a = sp.Q.from_dense(rng.standard_normal((48, 48)))
        b = sp.Q.from_dense(rng.standard_normal((48, 48)))
        err, budget = sp.M.multiply_error(a, b, sp.M.SpammConfig(tau=0.0))
        assert budget == 0.0 and err <= 1e-13 * sp.Q.node_norm(a) * sp.Q.node_norm(b)

    def test_error_bound_random_decay_pairs(self, sp):
        """test_multiply.py:182-198 -- ||C~ - C|| <= budget + 1e-12 ||A|| ||B||
        over 100 random decay pairs and six tau."""
        rng = np.random.default_rng(7)
        for _ in range(100):
            n = int(rng.integers(8, 49))
            alpha = float(rng.uniform(0.2, 2.5))
            ix = np.arange(n)
            dec = np.exp(-alpha * np.abs(ix[:, None] - ix[None, :]))
            a = sp.Q.from_dense(dec * rng.standard_normal((n, n)))
            b = sp.Q.from_dense(dec * rng.standard_normal((n, n)))
            slack = 1e-12 * sp.Q.node_norm(a) * sp.Q.node_norm(b)
            exact = sp.Q.to_dense(sp.M.exact_multiply(a, b))
            for tau in (1e-2, 1e-4, 1e-6, 1e-8, 1e-10, 1e-12):
                c, st = sp.M.spamm(a, b, sp.M.SpammConfig(tau=tau))
                assert float(np.linalg.norm(sp.Q.to_dense(c) - exact)) <= st.omitted_budget + slack

    def test_error_sweep_decreases_with_tau(self, sp):
        """test_multiply.py:201-210."""
        a = sp.G.gen_exponential(512, 1.0)
        b = sp.G.gen_exponential(512, 2.0)
        exact = sp.Q.to_dense(sp.M.exact_multiply(a, b))
        err = {}
        for tau in (1e-2, 1e-4, 1e-6, 1e-8, 1e-10):
            c, st = sp.M.spamm(a, b, sp.M.SpammConfig(tau=tau))
            err[tau] = float(np.linalg.norm(sp.Q.to_dense(c) - exact))
            assert err[tau] <= st.omitted_budget + 1e-12
        assert err[1e-10] < err[1e-2]

    def test_monotone_work_in_tau(self, sp):
        """test_multiply.py:213-219."""
        a = sp.G.gen_exponential(256, 0.7)
        b = sp.G.gen_exponential(256, 1.3)
        work = [sp.M.spamm(a, b, sp.M.SpammConfig(tau=t))[1].leaf_matmuls
                for t in (0.0, 1e-12, 1e-9, 1e-6, 1e-3, 1e-1)]
        assert all(x >= y for x, y in zip(work, work[1:]))

    def test_determinism_bit_identical(self, sp):
        """test_multiply.py:222-229 -- C bytes and ProductStats identical across runs."""
        a = sp.G.gen_exponential(256, 0.9)
        b = sp.G.gen_exponential(256, 1.1)
        cfg = sp.M.SpammConfig(tau=1e-7, collect_boxes=True)
        c1, s1 = sp.M.spamm(a, b, cfg)
        c2, s2 = sp.M.spamm(a, b, cfg)
        assert sp.Q.to_dense(c1).tobytes() == sp.Q.to_dense(c2).tobytes()
        assert s1 == s2

    def test_tiling_with_empty_skips(self, sp):
        """test_multiply.py:232-240 -- identity x identity at tau = 0."""
        i64 = sp.Q.identity(64)
        _, st = sp.M.spamm(i64, i64, sp.M.SpammConfig(tau=0.0))
        assert (st.leaf_matmuls, st.omitted_budget, st.pruned_volume) == (16, 0.0, 0)
        assert st.empty_skip_volume > 0 and st.covered_volume(4) == 64 ** 3

    def test_tier_tau_decay_is_more_conservative(self, sp):
        """test_multiply.py:243-250."""
        a = sp.G.gen_exponential(256, 0.7)
        b = sp.G.gen_exponential(256, 1.3)
        flat = sp.M.spamm(a, b, sp.M.SpammConfig(tau=1e-6))[1]
        dec = sp.M.spamm(a, b, sp.M.SpammConfig(tau=1e-6, tier_tau_decay=True))[1]
        assert dec.leaf_matmuls >= flat.leaf_matmuls
        assert dec.omitted_budget <= flat.omitted_budget
        assert dec.covered_volume(4) == a.padded_dim ** 3

    def test_submultiplicativity_identity(self, sp):
        """test_multiply.py:255-256."""
        assert sp.M.norm_submultiplicativity_check(sp.Q.identity(16), sp.Q.identity(16))

    def test_submultiplicativity_random_pairs(self, sp):
        """test_multiply.py:259-264."""
        rng = np.random.default_rng(8)
        for _ in range(100):
            a = sp.Q.from_dense(rng.standard_normal((32, 32)))
            b = sp.Q.from_dense(rng.standard_normal((32, 32)))
            assert sp.M.norm_submultiplicativity_check(a, b)

    def test_submultiplicativity_rank1_equality(self, sp):
        """test_multiply.py:267-277 -- rank-1 operands reach the bound to 1e-13."""
        rng = np.random.default_rng(9)
        u, v, w = (x / np.linalg.norm(x) for x in rng.standard_normal((3, 32)))
        a = sp.Q.from_dense(np.outer(u, v))
        b = sp.Q.from_dense(np.outer(v, w))
        assert sp.M.norm_submultiplicativity_check(a, b)
        got = sp.Q.node_norm(sp.M.exact_multiply(a, b))
        assert abs(got - sp.Q.node_norm(a) * sp.Q.node_norm(b)) <= 1e-13

    def test_box_log_roundtrip_and_order(self, sp, tmp_path):
        """test_multiply.py:292-308 -- the box log round-trips, is in Morton
        order of the lower corners, and every box is aligned to its edge."""
        a = sp.G.gen_exponential(128, 1.0)
        b = sp.G.gen_exponential(128, 2.0)
        _, st = sp.M.spamm(a, b, sp.M.SpammConfig(tau=1e-6, collect_boxes=True))
        assert st.boxes
        path = tmp_path / "boxes.log"
        sp.M.write_box_log(st.boxes, path, a.padded_dim)
        back = sp.M.read_box_log(path)
        assert sorted(map(repr, back)) == sorted(map(repr, st.boxes))
        keys = [morton3(x.i_lo, x.j_lo, x.k_lo) for x in back]
        assert keys == sorted(keys)
        for line in path.read_text().splitlines():
            tier, i0, j0, k0, edge = map(int, line.split())
            assert edge == a.padded_dim >> tier
            assert i0 % edge == 0 and j0 % edge == 0 and k0 % edge == 0

    @pytest.mark.parametrize("tau", [-1e-9, float("nan"), float("inf")])
    def test_config_rejects_bad_tau(self, sp, tau):
        """test_multiply.py:311-317."""
        with pytest.raises(ValueError):
            sp.M.SpammConfig(tau=tau)

    def test_dimension_mismatch_rejected(self, sp):
        """test_multiply.py:320-328 -- different n, or different leaf sizes."""
        rng = np.random.default_rng(10)
        a = sp.Q.from_dense(rng.standard_normal((16, 16)))
        with pytest.raises(sp.Q.DimensionMismatchError):
            sp.M.spamm(a, sp.Q.from_dense(rng.standard_normal((32, 32))), sp.M.SpammConfig())
        with pytest.raises(sp.Q.DimensionMismatchError):
            sp.M.spamm(a, sp.Q.from_dense(rng.standard_normal((16, 16)), leaf_size=2),
                       sp.M.SpammConfig())


# --------------------------------------- pkg/tests/test_acceptance.py:31-100
class TestAcceptance:
    def test_exact_product_matches_oracle(self, sp):
        """test_acceptance.py:31-52 -- 200 random pairs (n = 1..40, 64, 128;
        leaf 1/2/4) against the triple loop: relative error <= 1e-13.  (The
        reference's 60 s wall-clock budget is asserted too.)"""
        import time

        t0 = time.perf_counter()
        rng = np.random.default_rng(2026)
        sizes = [(q % 40) + 1 for q in range(188)] + [64] * 8 + [128] * 4
        worst = 0.0
        for q, (n, leaf) in enumerate(zip(sizes, itertools.cycle((1, 2, 4)))):
            ad, bd = rng.standard_normal((n, n)), rng.standard_normal((n, n))
            got = sp.Q.to_dense(sp.M.exact_multiply(sp.Q.from_dense(ad, leaf_size=leaf),
                                                    sp.Q.from_dense(bd, leaf_size=leaf)))
            ref = triple_loop(ad, bd)
            den = np.linalg.norm(ref)
            err = np.linalg.norm(got - ref) / (den if den > 0 else 1.0)
            assert err <= 1e-13, (q, n, leaf, err)
            worst = max(worst, err)
        assert time.perf_counter() - t0 < 60.0

    def test_truncation_error_bounded(self, sp):
        """test_acceptance.py:55-80 -- exponential and algebraic pairs at n = 512:
        error <= budget + 1e-12 ||A|| ||B|| for tau = 1e-2 .. 1e-10, and the
        error at 1e-10 is below the error at 1e-2."""
        pairs = {"exponential": (sp.G.gen_exponential(512, 1.0), sp.G.gen_exponential(512, 2.0)),
                 "algebraic": (sp.G.gen_algebraic(512, 3.0), sp.G.gen_algebraic(512, 3.0))}
        for label, (a, b) in pairs.items():
            exact = sp.Q.to_dense(sp.M.exact_multiply(a, b))
            slack = 1e-12 * sp.Q.node_norm(a) * sp.Q.node_norm(b)
            err = {}
            for tau in (1e-2, 1e-4, 1e-6, 1e-8, 1e-10):
                c, st = sp.M.spamm(a, b, sp.M.SpammConfig(tau=tau))
                err[tau] = float(np.linalg.norm(sp.Q.to_dense(c) - exact))
                assert err[tau] <= st.omitted_budget + slack, (label, tau)
            assert err[1e-10] < err[1e-2], label

    def test_product_space_tiling(self, sp):
        """test_acceptance.py:83-100 -- visited leaf cells + pruned boxes tile
        [0, 512)^3 exactly; no Empty skips; boxes aligned."""
        a = sp.G.gen_exponential(512, 1.0)
        b = sp.G.gen_exponential(512, 2.0)
        _, st = sp.M.spamm(a, b, sp.M.SpammConfig(tau=1e-8, collect_boxes=True))
        vol = sum(x.edge ** 3 for x in st.boxes)
        assert st.empty_skip_volume == 0 and vol == st.pruned_volume
        assert st.leaf_matmuls * 4 ** 3 + vol == 512 ** 3
        for x in st.boxes:
            assert x.edge == 512 >> x.tier
            assert x.i_lo % x.edge == 0 and x.j_lo % x.edge == 0 and x.k_lo % x.edge == 0

