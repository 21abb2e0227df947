"""Host-side checks of the §8(f3)/(f4) rows: Morton keys, MatrixMarket I/O,
box-log parsing and the generators' distance tables, against fixtures the
reference itself produced (tests/golden/make_io_golden.py).  No GPU."""

from __future__ import annotations

import gzip
import itertools
import os

import numpy as np
import pytest

from paper_1011_3534_b200 import matrixmarket as mm
from paper_1011_3534_b200.multiply import PrunedBox, read_box_log
from paper_1011_3534_b200.ordering import MortonKey, _interleave3, morton_key, split_key_ranges

IO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def golden():
    return np.load(os.path.join(IO, "io_golden.npz"))


def interleave_bits(i, j, k):
    """Independent restatement of ordering.py:24-34: bit b of i, j, k to
    3b+2, 3b+1, 3b."""
    key = 0
    for bit in range(22):
        key |= ((i >> bit) & 1) << (3 * bit + 2)
        key |= ((j >> bit) & 1) << (3 * bit + 1)
        key |= ((k >> bit) & 1) << (3 * bit)
    return key


# ----------------------------------------------------------------- Morton keys

def test_interleave_matches_bit_restatement():
    rng = np.random.default_rng(0)
    for i, j, k in rng.integers(0, 1 << 21, size=(500, 3)):
        assert _interleave3(i, j, k) == interleave_bits(int(i), int(j), int(k))
    assert _interleave3(0, 0, 0) == 0
    with pytest.raises(ValueError):
        _interleave3(-1, 0, 0)


def test_morton_key_units_and_origin():
    assert morton_key(PrunedBox(0, 0, 0, 8, 0), 8) == MortonKey(0, 0)
    assert morton_key(PrunedBox(1, 0, 0, 1, 3), 8).key == 4
    assert morton_key(PrunedBox(0, 1, 0, 1, 3), 8).key == 2
    assert morton_key(PrunedBox(0, 0, 1, 1, 3), 8).key == 1
    assert morton_key(PrunedBox(4, 4, 4, 4, 1), 8) == MortonKey(7, 1)
    with pytest.raises(ValueError):
        morton_key(PrunedBox(0, 0, 0, 4, 3), 8)


def test_morton_sort_visits_z_curve():
    def z(order):
        if order == 0:
            return [(0, 0, 0)]
        h = 1 << (order - 1)
        return [(a * h + x, b * h + y, c * h + w)
                for a, b, c in itertools.product((0, 1), repeat=3) for x, y, w in z(order - 1)]

    boxes = [PrunedBox(i, j, k, 1, 3) for i in range(8) for j in range(8) for k in range(8)]
    boxes.sort(key=lambda bx: morton_key(bx, 8).key)
    assert [(b.i_lo, b.j_lo, b.k_lo) for b in boxes] == z(3)


def test_split_key_ranges():
    r = split_key_ranges(np.arange(17), 5)
    assert r[0][0] == 0 and r[-1][1] == 17
    sizes = [b - a for a, b in r]
    assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    assert all(r[p][1] == r[p + 1][0] for p in range(4))
    assert split_key_ranges(np.arange(2), 4) == [(0, 1), (1, 2), (2, 2), (2, 2)]
    assert split_key_ranges([], 2) == [(0, 0), (0, 0)]
    with pytest.raises(ValueError):
        split_key_ranges(np.arange(3), 0)
    with pytest.raises(ValueError):
        split_key_ranges(np.array([2, 1]), 2)


# ------------------------------------------------------------------- box logs

def _log_lines(name):
    path = os.path.join(IO, name)
    if name.endswith(".gz"):
        with gzip.open(path, "rt") as fh:
            return fh.read().splitlines()
    return open(path).read().splitlines()


@pytest.mark.parametrize("name,n_pad", [("boxlog_exp128.txt", 128), ("boxlog_l16_b4.txt.gz", 512)])
def test_reference_box_logs_are_morton_sorted(name, n_pad, tmp_path):
    lines = _log_lines(name)
    assert len(lines) == int(golden()[name.split(".")[0] + "_n"])
    path = tmp_path / "log.txt"
    path.write_text("\n".join(lines) + "\n\n")      # trailing blank line is skipped
    boxes = read_box_log(path)
    assert len(boxes) == len(lines)
    keys = [interleave_bits(b.i_lo, b.j_lo, b.k_lo) for b in boxes]
    assert keys == sorted(keys) and len(set(keys)) == len(keys)
    for b in boxes:
        assert b.edge == n_pad >> b.tier
        assert b.i_lo % b.edge == b.j_lo % b.edge == b.k_lo % b.edge == 0
        assert morton_key(b, n_pad).tier == b.tier


def test_read_box_log_rejects_malformed(tmp_path):
    p = tmp_path / "bad.txt"
    p.write_text("1 2 3\n")
    with pytest.raises(ValueError):
        read_box_log(p)


# ---------------------------------------------------------------- MatrixMarket

@pytest.mark.parametrize("fmt,name", [("array", "mm_array.mtx"), ("coordinate", "mm_coord.mtx")])
def test_matrix_market_writer_bytes_match_reference(fmt, name, tmp_path):
    m = golden()["mm_matrix"]
    out = tmp_path / name
    mm.write_matrix_market(m, out, fmt=fmt)
    assert out.read_bytes() == open(os.path.join(IO, name), "rb").read()


@pytest.mark.parametrize("name", ["mm_array.mtx", "mm_coord.mtx"])
def test_matrix_market_reader_round_trip_bit_exact(name):
    m = golden()["mm_matrix"]
    back = mm.read_matrix_market(os.path.join(IO, name))
    assert back.dtype == np.float64 and back.shape == m.shape
    # bit-exact except the coordinate file drops the (negative) zeros
    if name == "mm_array.mtx":
        assert np.array_equal(back.view(np.int64), m.view(np.int64))
    else:
        assert np.array_equal(back, m)


def test_matrix_market_symmetric_and_comments(tmp_path):
    p = tmp_path / "sym.mtx"
    p.write_text("%%MatrixMarket matrix array real symmetric\n% comment\n\n3 3\n"
                 "1\n2\n3\n4 5\n6\n")
    got = mm.read_matrix_market(p)
    want = np.array([[1, 2, 3], [2, 4, 5], [3, 5, 6]], dtype=float)
    assert np.array_equal(got, want)
    p.write_text("%%MatrixMarket matrix coordinate integer symmetric\n3 3 3\n"
                 "1 1 2\n3 1 -1\n3 1 0.5\n")
    got = mm.read_matrix_market(p)
    want = np.zeros((3, 3))
    want[0, 0] = 2
    want[2, 0] = want[0, 2] = -0.5
    assert np.array_equal(got, want)


@pytest.mark.parametrize("text", [
    "%%Matrix matrix array real general\n1 1\n1\n",
    "%%MatrixMarket matrix array real\n1 1\n1\n",
    "%%MatrixMarket vector array real general\n1 1\n1\n",
    "%%MatrixMarket matrix list real general\n1 1\n1\n",
    "%%MatrixMarket matrix array complex general\n1 1\n1\n",
    "%%MatrixMarket matrix array real hermitian\n1 1\n1\n",
    "%%MatrixMarket matrix array real general\n",
    "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n",
    "%%MatrixMarket matrix array real symmetric\n2 2\n1\n2\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n",
])
def test_matrix_market_reader_errors(text, tmp_path):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(ValueError):
        mm.read_matrix_market(p)


def test_matrix_market_writer_errors(tmp_path):
    with pytest.raises(ValueError):
        mm.write_matrix_market(np.zeros(3), tmp_path / "x.mtx")
    with pytest.raises(ValueError):
        mm.write_matrix_market(np.zeros((2, 2)), tmp_path / "x.mtx", fmt="dense")


# ------------------------------------------------------- generator tables

def _expand(table, n, n_pad):
    i = np.arange(n)
    out = np.zeros((n_pad, n_pad))
    out[:n, :n] = table[np.abs(i[:, None] - i[None, :])]
    return out


@pytest.mark.parametrize("name", ["exp_n100_a0.3_b4", "exp_n257_a1.7_b8", "exp_n64_a0.05_b16",
                                  "alg_n100_p1.5_b4", "alg_n130_p0.7_b2", "alg_n64_p3_b8"])
def test_generator_distance_tables_reproduce_reference(name):
    """The host half of gen_exponential / gen_algebraic: the n-entry distance
    table expanded as the device does reproduces the reference's padded
    array bit for bit."""
    kind, n_s, par_s, _ = name.split("_")
    n, par = int(n_s[1:]), float(par_s[1:])
    want = golden()[f"gen_{name}_padded"]
    if kind == "exp":
        table = np.exp(-par * np.arange(n))
    else:
        table = np.zeros(n)
        table[1:] = np.arange(1, n, dtype=np.float64) ** (-par)
    got = _expand(table, n, want.shape[0])
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


def test_model_hamiltonian_validation():
    from paper_1011_3534_b200.generators import ModelHamiltonian

    assert ModelHamiltonian(10).n_occ == 5
    for kw in ({"n": 1}, {"n": 4, "kind": "metal"}, {"n": 4, "gap": 0.0},
               {"n": 4, "n_occ": 5}):
        with pytest.raises(ValueError):
            ModelHamiltonian(**kw)
