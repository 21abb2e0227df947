"""The reference's test-matrix generators, built on the device (generators.py:24-88).

Each matrix depends on |i - j| (or is tridiagonal), so it is fully described
by n numbers.  Those are evaluated on the host with exactly the numpy
expressions the reference applies to its n x n distance matrix -- elementwise
ufuncs, so each table entry equals the reference's entry at that distance --
and the N^2 expansion is written straight into the tree's device storage
(csrc/generate.cu) before K1 builds the pyramid.  The trees are therefore
bit-identical to the reference's ``from_dense`` of its dense array, without
an n x n host array or transfer.

The decay-profile analysis helpers of the reference module (positions,
``decay_profile``, fits, CSV) are reporting tools outside the multiply's
path and are not part of this package.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .quadtree import _wrap, get_device


def _dtype_code(dtype):
    target = np.dtype(np.float64 if dtype is None else dtype)
    if target == np.float64:
        return _lib.DTYPE_F64
    if target == np.float32:
        return _lib.DTYPE_F32
    raise ValueError(f"unsupported element dtype {target}")


def _toeplitz(table, n, leaf_size, dtype, device):
    table = np.ascontiguousarray(table, dtype=np.float64)
    h = ctypes.c_void_p()
    dev = get_device() if device is None else int(device)
    _lib.check(_lib.load().spamm_tree_toeplitz(table.ctypes.data, int(n), int(leaf_size),
                                               _dtype_code(dtype), dev, ctypes.byref(h)))
    return _wrap(h.value)


def gen_exponential(n, alpha, leaf_size=4, dtype=None, device=None):
    """Quadtree matrix with entries exp(-alpha |i - j|), alpha > 0
    (generators.py:24-30)."""
    if alpha <= 0:
        raise ValueError(f"alpha must be > 0, got {alpha}")
    dist = np.arange(max(int(n), 0))           # the distinct values of |i - j|
    return _toeplitz(np.exp(-alpha * dist), n, leaf_size, dtype, device)


def gen_algebraic(n, p, leaf_size=4, dtype=None, device=None):
    """Quadtree matrix with entries |i - j|^-p off the diagonal and 0 on it
    (generators.py:33-43)."""
    if p <= 0:
        raise ValueError(f"p must be > 0, got {p}")
    table = np.zeros(max(int(n), 0))
    dist = np.arange(1, max(int(n), 1), dtype=np.float64)
    table[1:] = dist ** (-float(p))
    return _toeplitz(table, n, leaf_size, dtype, device)


@dataclass
class ModelHamiltonian:
    """A 1-D tight-binding chain (generators.py:46-73): "gapped" alternates
    on-site energies +gap/2, -gap/2 with nearest-neighbour hopping;
    "gapless" is the uniform chain.  n_occ defaults to half filling."""

    n: int
    kind: str = "gapped"
    gap: float = 1.0
    hopping: float = 1.0
    n_occ: float | None = None

    def __post_init__(self):
        if self.n < 2:
            raise ValueError(f"n must be >= 2, got {self.n}")
        if self.kind not in ("gapped", "gapless"):
            raise ValueError(f"kind must be 'gapped' or 'gapless', got {self.kind!r}")
        if self.kind == "gapped" and self.gap <= 0:
            raise ValueError(f"gap must be > 0, got {self.gap}")
        if self.n_occ is None:
            self.n_occ = self.n // 2
        if not 0 <= self.n_occ <= self.n:
            raise ValueError(f"n_occ must be in [0, {self.n}], got {self.n_occ}")


def gen_model_hamiltonian(model, leaf_size=4, dtype=None, device=None):
    """The chain's Hamiltonian as a quadtree matrix (generators.py:76-88)."""
    n = model.n
    off = np.full(n - 1, model.hopping, dtype=np.float64)
    if model.kind == "gapped":
        sites = np.arange(n)
        diag = np.where(sites % 2 == 0, 0.5 * model.gap, -0.5 * model.gap).astype(np.float64)
    else:
        diag = np.zeros(n)
    h = ctypes.c_void_p()
    dev = get_device() if device is None else int(device)
    _lib.check(_lib.load().spamm_tree_tridiagonal(diag.ctypes.data, off.ctypes.data, int(n),
                                                  int(leaf_size), _dtype_code(dtype), dev,
                                                  ctypes.byref(h)))
    return _wrap(h.value)


__all__ = ["ModelHamiltonian", "gen_algebraic", "gen_exponential", "gen_model_hamiltonian"]
