"""The synthetic BASELINE.json inputs follow SURVEY.md §8(d) exactly."""

import numpy as np

from paper_1011_3534_b200 import workloads


def test_exponential_formula():
    n = 64
    a = workloads.exponential_decay(n, 0.9, 0)
    u = np.random.default_rng(0).uniform(-1.0, 1.0, size=(n, n))
    d = np.abs(np.arange(n)[:, None] - np.arange(n)[None, :]).astype(float)
    assert np.array_equal(a, u * np.power(0.9, d))
    s = workloads.exponential_decay(n, 0.95, 0, symmetric=True)
    assert np.array_equal(s, s.T)


def test_algebraic_formula():
    n = 48
    a = workloads.algebraic_decay(n, 3.0, 1)
    u = np.random.default_rng(1).uniform(-1.0, 1.0, size=(n, n))
    d = np.abs(np.arange(n)[:, None] - np.arange(n)[None, :]).astype(float)
    ref = u / (np.power(d, 3.0) + 1.0)
    assert np.array_equal(a, 0.5 * (ref + ref.T))


def test_configs_shapes():
    for name, cfg in workloads.CONFIGS.items():
        assert cfg["n"] in (1024, 4096, 8192, 65536)
        assert cfg["leaf"] in (32, 64)
        assert all(t > 0 for t in cfg["taus"])
