"""Seeded synthetic inputs for the BASELINE.json configs.

The reference publishes no dataset: every config is a synthetic decay matrix
defined by formula, so these generators stand in for the inputs exactly.
Recipe (the same arrays feed the CPU oracle and the GPU path):

* u = numpy PCG64 ``default_rng(seed).uniform(-1.0, 1.0, size=(n, n))``
* d = |i - j| as float64
* exponential decay ``u * lam**d``; algebraic decay ``u / (d**lam + 1)``
* symmetrisation ``0.5 * (A + A.T)``

Seeds: 0 for A, 1 for an independent B (BASELINE.json pins seeds for
config 1 only; SURVEY.md §8(d) states the same choice for the others).
Host-side numpy only -- input preparation, not the hot path.
"""

from __future__ import annotations

import numpy as np


def _distance(n):
    idx = np.arange(n, dtype=np.float64)
    return np.abs(idx[:, None] - idx[None, :])


def uniform(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, n))


def exponential_decay(n, lam, seed, symmetric=False):
    """A_ij = u_ij * lam**|i-j| (BASELINE.json configs 1, 2, 5)."""
    a = uniform(n, seed) * np.power(lam, _distance(n))
    return 0.5 * (a + a.T) if symmetric else a


def algebraic_decay(n, lam, seed, symmetric=True):
    """A_ij = u_ij / (|i-j|**lam + 1) (BASELINE.json config 3)."""
    a = uniform(n, seed) / (np.power(_distance(n), lam) + 1.0)
    return 0.5 * (a + a.T) if symmetric else a


# name -> (n, leaf, taus, builder returning (A, B))
CONFIGS = {
    "c1": dict(n=1024, leaf=32, taus=(1e-6,),
               make=lambda: (exponential_decay(1024, 0.9, 0), exponential_decay(1024, 0.9, 1))),
    "c2": dict(n=4096, leaf=64, taus=(1e-4, 1e-6, 1e-8, 1e-10),
               make=lambda: (lambda a: (a, a))(exponential_decay(4096, 0.95, 0, symmetric=True))),
    "c3_l2": dict(n=8192, leaf=64, taus=(1e-6, 1e-8),
                  make=lambda: (algebraic_decay(8192, 2.0, 0), algebraic_decay(8192, 2.0, 1))),
    "c3_l3": dict(n=8192, leaf=64, taus=(1e-6, 1e-8),
                  make=lambda: (algebraic_decay(8192, 3.0, 0), algebraic_decay(8192, 3.0, 1))),
    "c5": dict(n=65536, leaf=64, taus=(1e-8,),
               make=lambda: (lambda a: (a, a))(exponential_decay(65536, 0.98, 0, symmetric=True))),
}


def make_config(name):
    cfg = CONFIGS[name]
    a, b = cfg["make"]()
    return a, b, cfg["leaf"], cfg["taus"]


# --------------------------------------------------- config 4: SP2 lattice
def interleave3(x, y, z, bits):
    """Morton index of lattice site (x, y, z), x-major in every 3-bit group
    (the reference's ordering._interleave3 convention, ordering.py:24-34)."""
    s = np.zeros_like(np.asarray(x), dtype=np.int64)
    for b in range(bits):
        s |= (((np.asarray(x) >> b) & 1) << (3 * b + 2)) | (((np.asarray(y) >> b) & 1) << (3 * b + 1)) \
            | ((np.asarray(z) >> b) & 1) << (3 * b)
    return s


def cubic_lattice_hamiltonian(L, seed=0, hopping=-1.0, onsite=0.5):
    """BASELINE config 4 / SURVEY.md §8(d): tight-binding Hamiltonian of an
    L x L x L periodic cubic lattice (L a power of two), sites ordered along
    the Morton curve (site s = interleave3(x, y, z), a bijection onto
    [0, L^3)), nearest-neighbour hopping -1 (assigned, so L = 2's coinciding
    neighbours are one bond), on-site energies default_rng(seed).uniform(
    -onsite, onsite, n) indexed by s.  Dense float64 (host)."""
    bits = int(L).bit_length() - 1
    assert 1 << bits == L, "L must be a power of two"
    n = L ** 3
    h = np.zeros((n, n))
    x, y, z = np.meshgrid(np.arange(L), np.arange(L), np.arange(L), indexing="ij")
    x, y, z = x.ravel(), y.ravel(), z.ravel()
    s = interleave3(x, y, z, bits)
    for dx, dy, dz in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
        t = interleave3((x + dx) % L, (y + dy) % L, (z + dz) % L, bits)
        h[s, t] = hopping
    h[np.arange(n), np.arange(n)] = np.random.default_rng(seed).uniform(-onsite, onsite, n)
    return h


def cubic_lattice_hamiltonian_device(L, device, seed=0, hopping=-1.0, onsite=0.5):
    """The same matrix built on the GPU (torch float64 tensor): the on-site
    draw is numpy's (n values), the n x n fill happens on the device."""
    import torch

    bits = int(L).bit_length() - 1
    n = L ** 3
    h = torch.zeros((n, n), dtype=torch.float64, device=device)
    x, y, z = np.meshgrid(np.arange(L), np.arange(L), np.arange(L), indexing="ij")
    x, y, z = x.ravel(), y.ravel(), z.ravel()
    s = torch.from_numpy(interleave3(x, y, z, bits)).to(device)
    for dx, dy, dz in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
        t = torch.from_numpy(interleave3((x + dx) % L, (y + dy) % L, (z + dz) % L, bits)).to(device)
        h[s, t] = hopping
    d = torch.from_numpy(np.random.default_rng(seed).uniform(-onsite, onsite, n)).to(device)
    idx = torch.arange(n, device=device)
    h[idx, idx] = d
    return h


# ------------------------------------------------------------ on-device inputs
# c5 (n = 65536) would need > 100 GB of host staging through numpy.  These
# generators build the same formulas on the GPU with torch's Philox stream
# (same distribution, different draw than numpy's PCG64), row block by row
# block, for measurement runs only; parity is pinned on the host recipe above.
DEVICE_CONFIGS = {
    "c5": dict(n=65536, leaf=64, taus=(1e-8,), lam=0.98, seed=0),
}


def exponential_decay_device(n, lam, seed, device, dtype=None, block=4096):
    """sym(u * lam**|i-j|) with u ~ U[-1, 1), built on `device` (torch tensor)."""
    import torch

    dtype = dtype or torch.float64
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    u = torch.empty((n, n), dtype=torch.float64, device=device)
    u.uniform_(-1.0, 1.0, generator=g)
    a = torch.empty((n, n), dtype=dtype, device=device)
    idx = torch.arange(n, device=device, dtype=torch.float64)
    for r0 in range(0, n, block):
        r1 = min(n, r0 + block)
        d = (idx[r0:r1, None] - idx[None, :]).abs_()
        a[r0:r1] = (0.5 * (u[r0:r1] + u[:, r0:r1].T) * torch.pow(lam, d)).to(dtype)
        del d
    del u
    return a


def make_config_device(name, device, dtype=None):
    cfg = DEVICE_CONFIGS[name]
    a = exponential_decay_device(cfg["n"], cfg["lam"], cfg["seed"], device, dtype)
    return a, a, cfg["leaf"], cfg["taus"]
