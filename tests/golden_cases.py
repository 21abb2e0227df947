"""Loader for the reference-generated fixtures in tests/golden/.

Inputs are regenerated from seeds (paper_1011_3534_b200.workloads) or read
from the fixture for small cases; see tests/golden/make_golden.py.
"""

from __future__ import annotations

import json
import os

import numpy as np

from paper_1011_3534_b200 import workloads

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def cases():
    with open(os.path.join(GOLDEN, "golden.json")) as fh:
        return json.load(fh)["cases"]


def case_names(max_n=None):
    return [c["name"] for c in cases() if max_n is None or c["n"] <= max_n]


def load(name):
    meta = next(c for c in cases() if c["name"] == name)
    z = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
    dt = np.float32 if meta["dtype"] == "float32" else np.float64
    if "a" in z:
        a, b = z["a"], z["b"]
    elif meta["recipe"] and meta["recipe"].startswith("workloads:"):
        a, b, _, _ = workloads.make_config(meta["recipe"].split(":")[1])
    else:  # the reference's exp(-alpha |i-j|) pair, alpha = 1 and 2
        d = np.abs(np.arange(meta["n"])[:, None] - np.arange(meta["n"])[None, :])
        a, b = np.exp(-1.0 * d), np.exp(-2.0 * d)
    if meta["same_operand"]:
        b = a
    return meta, z, a.astype(dt, copy=False), b if b is a else b.astype(dt, copy=False)


# ------------------------------------------------ C block hashes (large cases)
HASH_SEED = 77


def hash_keys(leaf):
    """Odd 64-bit multipliers, one per element of a leaf block."""
    rng = np.random.default_rng(HASH_SEED)
    return rng.integers(0, 2 ** 63, size=leaf * leaf, dtype=np.uint64) * np.uint64(2) + np.uint64(1)


def block_hash(blocks):
    """h = sum_e bits(x_e) * K_e mod 2^64 per block of an (m, b, b) array:
    a change of any element's bits changes h (every K_e is odd).  The same
    function pins the reference's C in tests/golden/make_golden.py."""
    m, b = blocks.shape[0], blocks.shape[1]
    bits = np.ascontiguousarray(blocks).view(np.uint32 if blocks.dtype == np.float32
                                             else np.uint64).reshape(m, b * b).astype(np.uint64)
    with np.errstate(over="ignore"):
        return (bits * hash_keys(b)[None, :]).sum(axis=1, dtype=np.uint64)


def tree_blocks(tree, ids):
    """The listed leaves (ids i * block_grid + j) of a device tree, copied to
    the host through the C ABI (spamm_tree_blocks_to_host)."""
    import ctypes

    from paper_1011_3534_b200 import _lib

    ids = np.ascontiguousarray(ids, dtype=np.int64)
    out = np.empty((len(ids), tree.leaf_size, tree.leaf_size), dtype=tree.dtype)
    if len(ids):
        _lib.check(_lib.load().spamm_tree_blocks_to_host(tree._handle, ids.ctypes.data, len(ids),
                                                         out.ctypes.data))
    return out


def tree_block_hashes(tree, ids, chunk=4096):
    """block_hash of the listed leaves of a device tree, read in chunks."""
    out = np.empty(len(ids), np.uint64)
    for s in range(0, len(ids), chunk):
        out[s:s + chunk] = block_hash(tree_blocks(tree, ids[s:s + chunk]))
    return out
