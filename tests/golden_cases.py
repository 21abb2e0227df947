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
