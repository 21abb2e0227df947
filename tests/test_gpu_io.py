"""§8(f3)/(f4) on the GPU: the device Morton sort behind write_box_log, box
logs byte-identical to the reference's, the device generators bit-identical
to the reference's matrices, audit_norm_cache and the norm-bound check
(golden files from tests/golden/make_io_golden.py, made by the reference)."""

from __future__ import annotations

import gzip
import os

import numpy as np
import pytest

import paper_1011_3534_b200 as sp
from paper_1011_3534_b200.multiply import PrunedBox, morton_order

pytestmark = pytest.mark.gpu

IO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


@pytest.fixture(scope="module")
def golden():
    return np.load(os.path.join(IO, "io_golden.npz"))


def interleave_bits(i, j, k):
    key = 0
    for bit in range(21):
        key |= ((i >> bit) & 1) << (3 * bit + 2)
        key |= ((j >> bit) & 1) << (3 * bit + 1)
        key |= ((k >> bit) & 1) << (3 * bit)
    return key


def host_order(arr):
    """Python's stable sorted() by the Morton key (the reference's sort)."""
    keys = [interleave_bits(int(r[0]), int(r[1]), int(r[2])) for r in arr]
    return np.array(sorted(range(len(keys)), key=keys.__getitem__), dtype=np.int64)


# ------------------------------------------------------------ device sort

@pytest.mark.parametrize("n,hi", [(0, 8), (1, 8), (2047, 1 << 21), (2048, 64), (2049, 1 << 21),
                                  (20000, 4), (60001, 1 << 12)])
def test_device_morton_order_is_stable_sorted(n, hi):
    rng = np.random.default_rng(n)
    arr = np.zeros((n, 5), np.int64)
    arr[:, :3] = rng.integers(0, hi, size=(n, 3))      # small ranges force equal keys
    arr[:, 3] = 1
    arr[:, 4] = rng.integers(0, 9, size=n)
    got = morton_order(arr)
    assert np.array_equal(got, host_order(arr))


def test_device_morton_order_rejects_out_of_range():
    arr = np.array([[1 << 21, 0, 0, 1, 0]], np.int64)
    with pytest.raises(ValueError):
        morton_order(arr)


# -------------------------------------------------------------- box logs

def _golden_log(name):
    path = os.path.join(IO, name)
    if name.endswith(".gz"):
        with gzip.open(path, "rb") as fh:
            return fh.read()
    return open(path, "rb").read()


def test_box_log_matches_reference_bytes(tmp_path, golden):
    a = sp.gen_exponential(128, 1.0)
    b = sp.gen_exponential(128, 2.0)
    _, st = sp.spamm(a, b, sp.SpammConfig(tau=1e-6, collect_boxes=True))
    assert len(st.boxes) == int(golden["boxlog_exp128_n"])
    path = tmp_path / "boxes.log"
    sp.write_box_log(st.boxes, path, a.padded_dim)
    assert path.read_bytes() == _golden_log("boxlog_exp128.txt")
    back = sp.read_box_log(path)
    assert sorted(map(repr, back)) == sorted(map(repr, st.boxes))


def test_box_log_deep_tree_matches_reference_bytes(tmp_path, golden):
    a = sp.gen_exponential(512, 0.4)
    b = sp.gen_algebraic(512, 2.5)
    _, st = sp.spamm(a, b, sp.SpammConfig(tau=1e-7, collect_boxes=True))
    assert len(st.boxes) == int(golden["boxlog_l16_b4_n"])
    path = tmp_path / "boxes.log"
    sp.write_box_log(st.boxes, path, a.padded_dim)
    assert path.read_bytes() == _golden_log("boxlog_l16_b4.txt.gz")


def test_box_log_empty_and_shuffled(tmp_path):
    path = tmp_path / "empty.log"
    sp.write_box_log([], path, 8)
    assert path.read_text() == "" and sp.read_box_log(path) == []
    a = sp.gen_exponential(256, 0.7, leaf_size=8)
    _, st = sp.spamm(a, a, sp.SpammConfig(tau=1e-5, collect_boxes=True))
    rng = np.random.default_rng(3)
    shuffled = [st.boxes[q] for q in rng.permutation(len(st.boxes))]
    p1, p2 = tmp_path / "a.log", tmp_path / "b.log"
    sp.write_box_log(st.boxes, p1, a.padded_dim)
    sp.write_box_log(shuffled, p2, a.padded_dim)
    assert p1.read_bytes() == p2.read_bytes()


# ------------------------------------------------------------- generators

GEN = {
    "exp_n100_a0.3_b4": lambda: sp.gen_exponential(100, 0.3),
    "exp_n257_a1.7_b8": lambda: sp.gen_exponential(257, 1.7, leaf_size=8),
    "exp_n64_a0.05_b16": lambda: sp.gen_exponential(64, 0.05, leaf_size=16),
    "alg_n100_p1.5_b4": lambda: sp.gen_algebraic(100, 1.5),
    "alg_n130_p0.7_b2": lambda: sp.gen_algebraic(130, 0.7, leaf_size=2),
    "alg_n64_p3_b8": lambda: sp.gen_algebraic(64, 3, leaf_size=8),
    "ham_gapped_n96_b4": lambda: sp.gen_model_hamiltonian(sp.ModelHamiltonian(96)),
    "ham_gapped_n37_g0.3_t-1.25_b4":
        lambda: sp.gen_model_hamiltonian(sp.ModelHamiltonian(37, gap=0.3, hopping=-1.25)),
    "ham_gapless_n50_b8":
        lambda: sp.gen_model_hamiltonian(sp.ModelHamiltonian(50, kind="gapless"), leaf_size=8),
}


@pytest.mark.parametrize("name", sorted(GEN))
def test_generators_match_reference(name, golden):
    t = GEN[name]()
    pad = golden[f"gen_{name}_padded"]
    assert np.array_equal(t._padded.view(np.uint64), pad.view(np.uint64))
    assert np.array_equal(t._pyramid()[2].view(np.uint64),
                          golden[f"gen_{name}_nsq"].view(np.uint64))


@pytest.mark.parametrize("n,alpha,leaf", [(1, 0.5, 1), (1000, 0.01, 32), (4096, 0.25, 64)])
def test_gen_exponential_matches_dense_formula(n, alpha, leaf):
    """Against the reference's own expression evaluated here (same numpy)."""
    i = np.arange(n)
    dense = np.exp(-alpha * np.abs(i[:, None] - i[None, :]))
    t = sp.gen_exponential(n, alpha, leaf_size=leaf)
    ref = sp.from_dense(dense, leaf_size=leaf)
    assert np.array_equal(t._padded.view(np.uint64), ref._padded.view(np.uint64))
    assert np.array_equal(t._pyramid()[2], ref._pyramid()[2])
    t32 = sp.gen_exponential(n, alpha, leaf_size=leaf, dtype=np.float32)
    r32 = sp.from_dense(dense, leaf_size=leaf, dtype=np.float32)
    assert np.array_equal(t32._padded.view(np.uint32), r32._padded.view(np.uint32))


def test_generator_validation():
    with pytest.raises(ValueError):
        sp.gen_exponential(8, 0.0)
    with pytest.raises(ValueError):
        sp.gen_algebraic(8, -1.0)
    with pytest.raises(ValueError):
        sp.gen_exponential(0, 1.0)
    with pytest.raises(ValueError):
        sp.gen_exponential(8, 1.0, leaf_size=3)


# ------------------------------------------------- audits and norm bounds

def test_audit_norm_cache_is_zero():
    a = sp.gen_exponential(300, 0.2, leaf_size=8)
    b = sp.gen_algebraic(300, 1.2, leaf_size=8)
    assert sp.audit_norm_cache(a) == 0.0
    c, _ = sp.spamm(a, b, sp.SpammConfig(tau=1e-6))
    assert sp.audit_norm_cache(c) == 0.0
    assert sp.audit_norm_cache(sp.add(a, c)) == 0.0
    f = sp.from_dense(np.random.default_rng(1).standard_normal((70, 70)), leaf_size=4,
                      dtype=np.float32)
    assert sp.audit_norm_cache(f) == 0.0


def test_norm_submultiplicativity_check():
    a = sp.gen_exponential(200, 0.3, leaf_size=8)
    b = sp.gen_model_hamiltonian(sp.ModelHamiltonian(200), leaf_size=8)
    assert sp.norm_submultiplicativity_check(a, b)
    assert sp.norm_submultiplicativity_check(b, b)
    with pytest.raises(sp.DimensionMismatchError):
        sp.norm_submultiplicativity_check(a, sp.gen_exponential(100, 0.3, leaf_size=8))


def test_write_matrix_market_from_tree(tmp_path):
    d = np.random.default_rng(5).standard_normal((33, 33))
    d[d < 0.5] = 0.0
    t = sp.from_dense(d, leaf_size=4)
    for fmt in ("array", "coordinate"):
        p1, p2 = tmp_path / f"t_{fmt}.mtx", tmp_path / f"d_{fmt}.mtx"
        sp.write_matrix_market(t, p1, fmt=fmt)
        sp.write_matrix_market(d, p2, fmt=fmt)
        assert p1.read_bytes() == p2.read_bytes()
        back = sp.read_matrix_market(p1)
        assert np.array_equal(back, d)
