"""numpy's pairwise float64 summation, restated in the oracle (and on the
GPU in csrc/traverse.cu), must equal ndarray.sum() bit for bit -- it is how
the reference accumulates omitted_budget per tier (multiply.py:197)."""

import numpy as np
import pytest

from oracle import oracle


@pytest.mark.parametrize("n", [0, 1, 5, 7, 8, 9, 15, 16, 127, 128, 129, 255, 256, 1000, 4097,
                               8191, 8192, 8193, 65537, 300001])
def test_pairwise_matches_numpy(n):
    rng = np.random.default_rng(n)
    for scale in (1.0, 1e-12):
        a = np.ascontiguousarray(rng.standard_normal(n) ** 2 * scale * 10.0 ** rng.uniform(-6, 6, n))
        got = oracle.lib().oracle_pairwise_sum(a.ctypes.data, n)
        assert got.hex() == float(a.sum()).hex(), n
