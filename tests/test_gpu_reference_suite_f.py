"""The reference's behavioural suite for the SURVEY §8(f) rows -- the TC2/SP2
driver, the generators, MatrixMarket I/O, the Morton box keys -- and the rest
of its acceptance file, run against the B200 package through the ``spamm``
import shim (paper_1011_3534_b200.compat), like tests/test_gpu_reference_
suite.py does for the quadtree / multiply files.

Each test restates one test of the reference package (file:line in its
docstring; same inputs, same assertions, same tolerances) and reaches the
library only through ``spamm.*`` imports.  /root/reference is not on the GPU
box, so the checks are restated rather than executed from there; the
independent oracles the reference's conftest provides (dense eigensolver
projector, plain-array TC2 recurrence: pkg/tests/conftest.py:36-60) are
rewritten below.

Covered: pkg/tests/test_purification.py (all 19), test_matrixmarket.py (all
7 functions, 11 cases), test_generators.py:23-133 (the 14 generator /
Hamiltonian tests; the decay-profile helpers are out of scope),
test_ordering.py:159-206 (the 4 Morton key / key-range tests; the Hilbert
atom ordering is out of scope), test_acceptance.py:103-203 (3; the matched-error
comparison pinned to the reference's results, see its docstring).
"""

import itertools
import os

import numpy as np
import pytest

from paper_1011_3534_b200 import compat

pytestmark = pytest.mark.gpu


class _NS:
    pass


@pytest.fixture(scope="module")
def sp():
    """The library's modules, imported under the reference's names."""
    compat.install()
    import spamm.generators as G
    import spamm.matrixmarket as MM
    import spamm.multiply as M
    import spamm.ordering as O
    import spamm.purification as P
    import spamm.quadtree as Q

    ns = _NS()
    ns.G, ns.MM, ns.M, ns.O, ns.P, ns.Q = G, MM, M, O, P, Q
    yield ns
    compat.uninstall()


# ----------------------------------------------------- independent oracles

def eig_projector(fd, n_occ):
    """Projector onto the n_occ lowest eigenvectors (dense eigensolver)."""
    vecs = np.linalg.eigh(fd)[1][:, :n_occ]
    return vecs @ vecs.T


def dense_tc2(fd, n_occ, sweeps=50):
    """Plain-array TC2: Gershgorin interval -> X0 = (hi I - F) / (hi - lo);
    per sweep X <- X^2 if Tr X >= n_occ else 2X - X^2; stops at the
    idempotency floor 16 eps n."""
    n = fd.shape[0]
    d = np.diag(fd)
    r = np.abs(fd).sum(axis=1) - np.abs(d)
    lo, hi = float((d - r).min()), float((d + r).max())
    if hi <= lo:
        return 0.5 * np.eye(n)
    x = (hi * np.eye(n) - fd) / (hi - lo)
    floor = 16.0 * np.finfo(np.float64).eps * n
    for _ in range(sweeps):
        sq = x @ x
        if np.linalg.norm(sq - x, "fro") <= floor:
            break
        x = sq if np.trace(x) >= n_occ else 2.0 * x - sq
    return x


def _gapped(sp, n, gap=1.0, hopping=1.0):
    return sp.G.gen_model_hamiltonian(sp.G.ModelHamiltonian(n, "gapped", gap=gap, hopping=hopping))


def _model256(sp, kind):
    n = 256
    f = sp.G.gen_model_hamiltonian(sp.G.ModelHamiltonian(n=n, kind=kind))
    out = {"n": n, "n_occ": n // 2, "tree": f,
           "exact": sp.P.purify(f, n // 2, sp.P.SpammMode(0.0))}
    if kind == "gapped":
        out["dense"] = f.to_dense()
        out["projector"] = eig_projector(out["dense"], n // 2)
    return out


@pytest.fixture(scope="module")
def gapped256(sp):
    """conftest.py:63-78: gapped chain at n = 256, its dense form, its
    eigenprojector and the exact-algebra purification."""
    return _model256(sp, "gapped")


@pytest.fixture(scope="module")
def gapless256(sp):
    """conftest.py:81-86."""
    return _model256(sp, "gapless")


# ======================================================= test_purification.py

def test_initial_guess_two_level(sp):
    """test_purification.py:30-32"""
    x0 = sp.P.tc2_initial_guess(sp.Q.from_dense(np.diag([-1.0, 1.0])))
    assert np.array_equal(sp.Q.to_dense(x0), np.diag([1.0, 0.0]))


def test_initial_guess_degenerate_interval(sp):
    """test_purification.py:35-37"""
    x0 = sp.P.tc2_initial_guess(sp.Q.from_dense(np.zeros((4, 4))))
    assert np.array_equal(sp.Q.to_dense(x0), 0.5 * np.eye(4))


def test_initial_guess_spectrum_in_unit_interval(sp):
    """test_purification.py:40-47"""
    d = np.random.default_rng(0).standard_normal((32, 32))
    d = d + d.T
    ev = np.linalg.eigvalsh(sp.Q.to_dense(sp.P.tc2_initial_guess(sp.Q.from_dense(d))))
    eps = np.finfo(np.float64).eps
    assert ev.min() >= -8 * eps and ev.max() <= 1 + 8 * eps


def test_step_fixed_point_both_branches(sp):
    """test_purification.py:52-56"""
    x = sp.Q.from_dense(np.diag([1.0, 0.0]))
    for n_occ in (1, 2):
        nxt, _ = sp.P.tc2_step(x, n_occ, sp.P.SpammMode(0.0))
        assert np.array_equal(sp.Q.to_dense(nxt), np.diag([1.0, 0.0]))


def test_step_squares_on_high_trace(sp):
    """test_purification.py:59-62"""
    nxt, _ = sp.P.tc2_step(sp.Q.from_dense(0.5 * np.eye(2)), 1, sp.P.SpammMode(0.0))
    assert np.array_equal(sp.Q.to_dense(nxt), 0.25 * np.eye(2))


def test_step_dropping_filters_resultant_only(sp):
    """test_purification.py:65-75"""
    rng = np.random.default_rng(1)
    idx = np.arange(32)
    d = np.exp(-0.8 * np.abs(idx[:, None] - idx[None, :])) * rng.uniform(0.5, 1.0, size=(32, 32))
    x = sp.Q.from_dense(d)
    tau = 1e-3
    nxt, _ = sp.P.tc2_step(x, 1, sp.P.DroppingMode(tau))
    expect = sp.Q.filter_drop(sp.M.exact_multiply(x, x), tau)
    assert np.array_equal(sp.Q.to_dense(nxt), sp.Q.to_dense(expect))


def test_step_converges_gapped64(sp):
    """test_purification.py:78-85"""
    x = sp.P.tc2_initial_guess(_gapped(sp, 64))
    for _ in range(50):
        x, _ = sp.P.tc2_step(x, 32, sp.P.SpammMode(0.0))
    x2 = sp.M.exact_multiply(x, x)
    assert np.linalg.norm(sp.Q.to_dense(x2) - sp.Q.to_dense(x)) <= 1e-10


def test_purify_two_level_analytic(sp):
    """test_purification.py:90-96"""
    f = sp.Q.from_dense(np.diag([-1.0, 1.0]))
    for mode in (sp.P.SpammMode(0.0), sp.P.SpammMode(1e-8), sp.P.DroppingMode(1e-8)):
        res = sp.P.purify(f, 1, mode)
        assert np.array_equal(sp.Q.to_dense(res.density), np.diag([1.0, 0.0]))
        assert res.energy == -1.0 and res.delta_e_rel == 0.0


def test_purify_matches_eigensolver_projector(sp, gapped256):
    """test_purification.py:99-101"""
    p = sp.Q.to_dense(gapped256["exact"].density)
    assert np.linalg.norm(p - gapped256["projector"]) <= 1e-8


def test_purify_idempotency_and_trace(sp, gapped256):
    """test_purification.py:104-109"""
    p = gapped256["exact"].density
    p2 = sp.M.exact_multiply(p, p)
    assert np.linalg.norm(sp.Q.to_dense(p2) - sp.Q.to_dense(p)) <= 1e-8 * gapped256["n"]
    assert abs(sp.Q.trace(p) - gapped256["n_occ"]) <= 1e-6


def test_purify_commutes_with_generator(sp, gapped256):
    """test_purification.py:112-116"""
    p = sp.Q.to_dense(gapped256["exact"].density)
    f = gapped256["dense"]
    assert np.linalg.norm(p @ f - f @ p) <= 1e-6 * np.linalg.norm(f)


def test_error_monotone_in_tau(sp, gapped256):
    """test_purification.py:119-126"""
    ref = gapped256["exact"].energy
    for mode_cls in (sp.P.SpammMode, sp.P.DroppingMode):
        tight = sp.P.purify(gapped256["tree"], 128, mode_cls(1e-12), reference_energy=ref)
        loose = sp.P.purify(gapped256["tree"], 128, mode_cls(1e-4), reference_energy=ref)
        assert tight.delta_e_rel <= loose.delta_e_rel


def test_matmul_accounting(sp):
    """test_purification.py:129-135"""
    res = sp.P.purify(_gapped(sp, 64), 32, sp.P.SpammMode(1e-6), max_iter=12)
    assert res.iterations == 12
    assert len(res.step_leaf_matmuls) == 12 and len(res.trace_history) == 13
    assert res.total_leaf_matmuls == sum(res.step_leaf_matmuls)
    assert res.avg_leaf_matmuls == res.total_leaf_matmuls / 12


def test_purify_tau0_reference_is_self(sp):
    """test_purification.py:138-141"""
    res = sp.P.purify(_gapped(sp, 64), 32, sp.P.SpammMode(0.0))
    assert res.delta_e_rel == 0.0 and res.reference_energy == res.energy


def test_match_returns_boundary_for_coarse_target(sp):
    """test_purification.py:146-151"""
    res = sp.P.match_error_threshold(_gapped(sp, 64), 32, 1e3, sp.P.SpammMode(0.0))
    assert res.hit_boundary and not res.converged and res.tau == 1e-1


def test_match_raises_below_error_floor(sp):
    """test_purification.py:154-157"""
    with pytest.raises(sp.P.ThresholdMatchError):
        sp.P.match_error_threshold(_gapped(sp, 64), 32, 1e-17, sp.P.SpammMode(0.0))


def test_match_verifies_on_rerun_gapped128(sp):
    """test_purification.py:160-168"""
    h = _gapped(sp, 128)
    ref = sp.P.purify(h, 64, sp.P.SpammMode(0.0)).energy
    res = sp.P.match_error_threshold(h, 64, 1e-7, sp.P.SpammMode(0.0), reference_energy=ref)
    assert res.converged
    check = sp.P.purify(h, 64, sp.P.SpammMode(res.tau), reference_energy=ref)
    assert 0.5e-7 <= check.delta_e_rel <= 2e-7


def test_purify_report_schema(sp, tmp_path):
    """test_purification.py:173-196"""
    res = sp.P.purify(_gapped(sp, 64), 32, sp.P.SpammMode(1e-7), max_iter=9)
    path = tmp_path / "report.csv"
    sp.P.write_purify_report(res, path)
    lines = path.read_text().splitlines()
    assert lines[0] == "iteration,trace,leaf_matmuls,cumulative_matmuls"
    assert len(lines) == 11
    running = 0
    for i, row in enumerate(lines[1:-1], start=1):
        it, tr, count, cumulative = row.split(",")
        running += int(count)
        assert int(it) == i and float(tr) == res.trace_history[i]
        assert int(count) == res.step_leaf_matmuls[i - 1] and int(cumulative) == running
    assert running == res.total_leaf_matmuls
    summary = lines[-1].split(",")
    assert summary[0] == "summary"
    fields = dict(tok.split("=") for tok in summary[1:])
    assert float(fields["energy"]) == res.energy
    assert float(fields["delta_e_rel"]) == res.delta_e_rel
    assert float(fields["avg_leaf_matmuls"]) == res.avg_leaf_matmuls


def test_purify_validation(sp):
    """test_purification.py:201-221"""
    P = sp.P
    asym = sp.Q.from_dense(np.random.default_rng(2).standard_normal((8, 8)))
    with pytest.raises(ValueError):
        P.purify(asym, 4, P.SpammMode(0.0))
    h = _gapped(sp, 8)
    for bad_occ in (-1, 9):
        with pytest.raises(ValueError):
            P.purify(h, bad_occ, P.SpammMode(0.0))
    with pytest.raises(ValueError):
        P.purify(h, 4, P.SpammMode(0.0), max_iter=0)
    with pytest.raises(ValueError):
        P.purify(h, 4, P.SpammMode(-1e-8))
    with pytest.raises(TypeError):
        P.tc2_step(P.tc2_initial_guess(h), 4, "spamm")
    with pytest.raises(ValueError):
        P.match_error_threshold(h, 4, 0.0, P.SpammMode(0.0))
    with pytest.raises(ValueError):
        P.match_error_threshold(h, 4, 1e-6, P.SpammMode(0.0), band_factor=1.0)


# ======================================================= test_matrixmarket.py

def _tricky_matrix():
    """test_matrixmarket.py:12-21: awkward doubles (1/3, a huge value, the
    smallest denormal and normal, an explicit zero)."""
    m = np.random.default_rng(0).standard_normal((7, 7))
    m[0, 0] = 0.1
    m[1, 2] = -1.0 / 3.0
    m[2, 1] = np.pi * 1e300
    m[3, 4] = 5e-324
    m[4, 3] = -2.2250738585072014e-308
    m[5, 5] = 0.0
    return m


@pytest.mark.parametrize("fmt", ["array", "coordinate"])
def test_mm_roundtrip_bit_exact(sp, fmt, tmp_path):
    """test_matrixmarket.py:24-30"""
    m = _tricky_matrix()
    path = tmp_path / f"m.{fmt}.mtx"
    sp.MM.write_matrix_market(m, path, fmt=fmt)
    assert sp.MM.read_matrix_market(path).tobytes() == m.tobytes()


@pytest.mark.parametrize("fmt", ["array", "coordinate"])
def test_mm_roundtrip_nonsquare_and_quadtree(sp, fmt, tmp_path):
    """test_matrixmarket.py:33-41"""
    rng = np.random.default_rng(1)
    rect = rng.standard_normal((3, 5))
    sp.MM.write_matrix_market(rect, tmp_path / "rect.mtx", fmt=fmt)
    assert sp.MM.read_matrix_market(tmp_path / "rect.mtx").tobytes() == rect.tobytes()
    square = rng.standard_normal((6, 6))
    sp.MM.write_matrix_market(sp.Q.from_dense(square), tmp_path / "tree.mtx", fmt=fmt)
    assert sp.MM.read_matrix_market(tmp_path / "tree.mtx").tobytes() == square.tobytes()


def test_mm_headers_and_zero_matrix(sp, tmp_path):
    """test_matrixmarket.py:44-55"""
    sp.MM.write_matrix_market(np.zeros((3, 3)), tmp_path / "za.mtx", fmt="array")
    lines = (tmp_path / "za.mtx").read_text().splitlines()
    assert lines[:2] == ["%%MatrixMarket matrix array real general", "3 3"]
    assert len(lines) == 2 + 9
    sp.MM.write_matrix_market(np.zeros((3, 3)), tmp_path / "zc.mtx", fmt="coordinate")
    lines = (tmp_path / "zc.mtx").read_text().splitlines()
    assert lines == ["%%MatrixMarket matrix coordinate real general", "3 3 0"]


@pytest.mark.parametrize("fmt", ["array", "coordinate"])
def test_mm_scipy_reads_our_files(sp, fmt, tmp_path):
    """test_matrixmarket.py:58-66"""
    scipy_io = pytest.importorskip("scipy.io")
    import scipy.sparse

    m = _tricky_matrix()
    path = tmp_path / "ours.mtx"
    sp.MM.write_matrix_market(m, path, fmt=fmt)
    got = scipy_io.mmread(path)
    if scipy.sparse.issparse(got):
        got = got.toarray()
    assert np.array_equal(np.asarray(got), m)


def test_mm_we_read_scipy_files(sp, tmp_path):
    """test_matrixmarket.py:69-83"""
    scipy_io = pytest.importorskip("scipy.io")
    import scipy.sparse

    dense = np.random.default_rng(2).standard_normal((5, 4))
    scipy_io.mmwrite(tmp_path / "sd.mtx", dense)
    assert np.allclose(sp.MM.read_matrix_market(tmp_path / "sd.mtx"), dense, rtol=0, atol=0)
    sparse = scipy.sparse.random(8, 8, density=0.2, random_state=3)
    scipy_io.mmwrite(tmp_path / "ss.mtx", sparse)
    assert np.array_equal(sp.MM.read_matrix_market(tmp_path / "ss.mtx"), sparse.toarray())
    sym = dense[:4, :4] + dense[:4, :4].T
    scipy_io.mmwrite(tmp_path / "sym.mtx", sym, symmetry="symmetric")
    assert np.array_equal(sp.MM.read_matrix_market(tmp_path / "sym.mtx"), sym)


def test_mm_symmetric_coordinate_mirrors_entries(sp, tmp_path):
    """test_matrixmarket.py:86-96"""
    path = tmp_path / "sym.mtx"
    path.write_text("%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n2 1 5.0\n3 3 7.0\n")
    expect = np.zeros((3, 3))
    expect[1, 0] = expect[0, 1] = 5.0
    expect[2, 2] = 7.0
    assert np.array_equal(sp.MM.read_matrix_market(path), expect)


def test_mm_read_rejects_malformed(sp, tmp_path):
    """test_matrixmarket.py:99-121"""
    texts = {
        "bad.mtx": "not a matrix market file\n1 1\n0\n",
        "cx.mtx": "%%MatrixMarket matrix array complex general\n1 1\n1.0 0.0\n",
        "short.mtx": "%%MatrixMarket matrix array real general\n2 2\n1.0\n",
    }
    for name, text in texts.items():
        (tmp_path / name).write_text(text)
        with pytest.raises(ValueError):
            sp.MM.read_matrix_market(tmp_path / name)
    with pytest.raises(ValueError):
        sp.MM.write_matrix_market(np.eye(2), tmp_path / "x.mtx", fmt="harwell")
    with pytest.raises(ValueError):
        sp.MM.write_matrix_market(np.zeros(3), tmp_path / "x.mtx")


# ========================================================= test_generators.py

def test_gen_exponential_spot_values(sp):
    """test_generators.py:23-27"""
    a = sp.Q.to_dense(sp.G.gen_exponential(512, 1.0))
    assert a[0, 0] == 1.0 and a[0, 1] == np.exp(-1.0) and a[17, 42] == np.exp(-25.0)


def test_gen_exponential_huge_alpha_is_identity(sp):
    """test_generators.py:30-34"""
    a = sp.Q.to_dense(sp.G.gen_exponential(64, 700.0))
    assert np.max(np.abs(a - np.eye(64))) <= 1e-300
    assert np.count_nonzero(sp.Q.to_dense(sp.G.gen_exponential(64, 800.0))) == 64


def test_gen_exponential_matches_formula(sp):
    """test_generators.py:37-41"""
    for n, alpha in ((30, 0.3), (512, 2.0)):
        idx = np.arange(n)
        ref = np.exp(-alpha * np.abs(idx[:, None] - idx[None, :]))
        assert np.array_equal(sp.Q.to_dense(sp.G.gen_exponential(n, alpha)), ref)


def test_gen_exponential_rejects_bad_alpha(sp):
    """test_generators.py:44-48"""
    for alpha in (0.0, -1.0):
        with pytest.raises(ValueError):
            sp.G.gen_exponential(16, alpha)


def test_gen_algebraic_values(sp):
    """test_generators.py:53-58"""
    a = sp.Q.to_dense(sp.G.gen_algebraic(512, 3.0))
    assert np.array_equal(np.diag(a), np.zeros(512))
    off = np.abs(np.arange(512)[:, None] - np.arange(512)[None, :]) == 1
    assert np.array_equal(a[off], np.ones(off.sum()))
    assert a[0, 2] == 0.125


def test_gen_algebraic_n2_any_p(sp):
    """test_generators.py:61-64"""
    for p in (0.5, 1.0, 3.0, 7.0):
        assert np.array_equal(sp.Q.to_dense(sp.G.gen_algebraic(2, p)),
                              np.array([[0.0, 1.0], [1.0, 0.0]]))


def test_gen_algebraic_rejects_bad_p(sp):
    """test_generators.py:67-71"""
    for p in (0.0, -2.0):
        with pytest.raises(ValueError):
            sp.G.gen_algebraic(16, p)


def test_generators_symmetric_bitexact(sp):
    """test_generators.py:74-77"""
    for m in (sp.G.gen_exponential(100, 0.8), sp.G.gen_algebraic(100, 3.0)):
        d = sp.Q.to_dense(m)
        assert np.array_equal(d, d.T)


def test_generator_roundtrip_exact(sp):
    """test_generators.py:80-83"""
    d = sp.Q.to_dense(sp.G.gen_exponential(75, 1.3))
    assert np.array_equal(sp.Q.to_dense(sp.Q.from_dense(d)), d)


def test_gapped_n2_zero_hopping_eigenvalues(sp):
    """test_generators.py:88-92"""
    h = sp.G.gen_model_hamiltonian(sp.G.ModelHamiltonian(2, "gapped", gap=2.0, hopping=0.0))
    d = sp.Q.to_dense(h)
    assert np.array_equal(d, np.diag([1.0, -1.0]))
    assert sorted(np.linalg.eigvalsh(d)) == [-1.0, 1.0]


def test_gapless_spectrum_matches_dense_oracle(sp):
    """test_generators.py:95-101"""
    n, t = 256, 1.0
    h = sp.Q.to_dense(sp.G.gen_model_hamiltonian(sp.G.ModelHamiltonian(n, "gapless", hopping=t)))
    k = np.arange(1, n + 1)
    ref = np.sort(2.0 * t * np.cos(k * np.pi / (n + 1)))
    assert np.max(np.abs(np.sort(np.linalg.eigvalsh(h)) - ref)) <= 1e-10


def test_gapped_spectral_gap_near_requested(sp):
    """test_generators.py:104-110"""
    n = 256
    ev = np.sort(np.linalg.eigvalsh(sp.Q.to_dense(_gapped(sp, n))))
    assert abs((ev[n // 2] - ev[n // 2 - 1]) - 1.0) <= 0.05


def test_hamiltonian_structure_and_symmetry(sp):
    """test_generators.py:113-119"""
    d = sp.Q.to_dense(sp.G.gen_model_hamiltonian(
        sp.G.ModelHamiltonian(10, "gapped", gap=0.6, hopping=2.5)))
    assert np.array_equal(d, d.T)
    assert d[3, 4] == 2.5 and d[4, 3] == 2.5
    assert d[0, 0] == 0.3 and d[1, 1] == -0.3 and d[2, 5] == 0.0


def test_hamiltonian_validation(sp):
    """test_generators.py:122-131"""
    H = sp.G.ModelHamiltonian
    for args, kw in (((1,), {}), ((8, "metallic"), {}), ((8, "gapped"), {"gap": -1.0}),
                     ((8,), {"n_occ": 9})):
        with pytest.raises(ValueError):
            H(*args, **kw)
    assert H(8).n_occ == 4


# ======================================================= test_ordering.py (Morton)

def test_morton_origin_and_units(sp):
    """test_ordering.py:159-163"""
    Box, key = sp.M.PrunedBox, sp.O.morton_key
    assert key(Box(0, 0, 0, 8, 0), 8) == sp.O.MortonKey(0, 0)
    assert key(Box(1, 0, 0, 1, 3), 8).key == 4
    assert key(Box(0, 1, 0, 1, 3), 8).key == 2
    assert key(Box(0, 0, 1, 1, 3), 8).key == 1


def _z_curve(order):
    if order == 0:
        return [(0, 0, 0)]
    half, sub = 1 << (order - 1), _z_curve(order - 1)
    return [(i * half + a, j * half + b, k * half + c)
            for i, j, k in itertools.product((0, 1), repeat=3) for a, b, c in sub]


def test_morton_sort_is_z_curve(sp):
    """test_ordering.py:176-181"""
    boxes = [sp.M.PrunedBox(i, j, k, 1, 3) for i in range(8) for j in range(8) for k in range(8)]
    boxes.sort(key=lambda bx: sp.O.morton_key(bx, 8).key)
    assert [(bx.i_lo, bx.j_lo, bx.k_lo) for bx in boxes] == _z_curve(3)


def test_morton_rejects_inconsistent_box(sp):
    """test_ordering.py:184-186"""
    with pytest.raises(ValueError):
        sp.O.morton_key(sp.M.PrunedBox(0, 0, 0, 4, 3), 8)


def test_split_key_ranges_balance_and_cover(sp):
    """test_ordering.py:191-203"""
    keys = np.arange(17)
    ranges = sp.O.split_key_ranges(keys, 5)
    assert ranges[0][0] == 0 and ranges[-1][1] == 17
    sizes = [hi - lo for lo, hi in ranges]
    assert max(sizes) - min(sizes) <= 1
    assert all(a[1] == b[0] for a, b in zip(ranges[:-1], ranges[1:]))
    assert sp.O.split_key_ranges(np.arange(2), 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    with pytest.raises(ValueError):
        sp.O.split_key_ranges(keys, 0)
    with pytest.raises(ValueError):
        sp.O.split_key_ranges(np.array([3, 1, 2]), 2)


# ================================================== test_acceptance.py:103-203

def test_near_linear_scaling_gapped_density(sp):
    """test_acceptance.py:103-136: self-products of purified gapped density
    matrices -- tau = 0 does exactly (n/4)^3 leaf products (8x per doubling),
    tau = 1e-8 approaches linear work (last doubling ratio <= 2.5)."""
    sizes = (256, 512, 1024, 2048)
    pruned, full = {}, {}
    for n in sizes:
        f = sp.G.gen_model_hamiltonian(sp.G.ModelHamiltonian(n=n, kind="gapped"))
        p = sp.Q.from_dense(dense_tc2(f.to_dense(), n // 2))
        pruned[n] = sp.M.spamm(p, p, sp.M.SpammConfig(tau=1e-8))[1].leaf_matmuls
        if n <= 1024:
            full[n] = sp.M.spamm(p, p, sp.M.SpammConfig(tau=0.0))[1].leaf_matmuls
            assert full[n] == (n // 4) ** 3
        del p, f
    assert full[512] / full[256] == 8.0 and full[1024] / full[512] == 8.0
    ratios = [pruned[b] / pruned[a] for a, b in zip(sizes, sizes[1:])]
    assert ratios[-1] <= 2.5, (ratios, pruned)


def test_purified_density_correctness(sp, gapped256):
    """test_acceptance.py:189-201"""
    p = sp.Q.to_dense(gapped256["exact"].density)
    f = gapped256["dense"]
    assert float(np.linalg.norm(p - gapped256["projector"])) <= 1e-8
    assert abs(sp.Q.trace(gapped256["exact"].density) - gapped256["n_occ"]) <= 1e-6
    assert float(np.linalg.norm(p @ f - f @ p)) <= 1e-6 * float(np.linalg.norm(f))


MATCH_GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "match_golden.json")


def test_matched_error_work_comparison(sp, gapped256, gapless256):
    """test_acceptance.py:139-186: the six matched-error searches (gapped
    1e-6 and 1e-8, gapless 1e-5; in-multiply pruning and drop-then-multiply;
    16 bisection steps).  The reference's own assertions on them (both modes
    inside the band, pruning never above dropping) FAIL on the reference
    itself -- run here, its gapless pruning search ends outside the band after
    18 evaluations and pruning averages more leaf products than dropping in
    all three cases -- so the drop-in is held to the reference's RESULTS
    instead (tests/golden/match_golden.json, written by tests/golden/
    make_match_golden.py from the real package): threshold, error, outcome,
    evaluation count, final energy and every sweep's leaf-product count, bit
    for bit, including the coarse thresholds whose iterates diverge."""
    import json

    with open(MATCH_GOLDEN) as fh:
        golden = json.load(fh)
    fxs = {"gapped": gapped256, "gapless": gapless256}
    for key, g in sorted(golden.items()):
        fx = fxs[g["kind"]]
        assert fx["exact"].energy == float.fromhex(g["exact_energy"]), key
        mode = sp.P.SpammMode(0.0) if g["mode"] == "spamm" else sp.P.DroppingMode(0.0)
        r = sp.P.match_error_threshold(fx["tree"], fx["n_occ"], g["target"], mode, max_steps=16,
                                       reference_energy=fx["exact"].energy)
        assert r.tau == float.fromhex(g["tau"]), key
        assert r.delta_e_rel == float.fromhex(g["delta_e_rel"]), key
        assert (r.converged, r.hit_boundary, r.evaluations) == \
            (g["converged"], g["hit_boundary"], g["evaluations"]), key
        assert r.result.energy == float.fromhex(g["energy"]), key
        assert r.result.total_leaf_matmuls == g["total_leaf_matmuls"], key
        assert list(r.result.step_leaf_matmuls) == g["step_leaf_matmuls"], key
