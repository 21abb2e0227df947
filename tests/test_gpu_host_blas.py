"""The 1e-12 contract bar against THIS host's BLAS.

tests/golden pins C to the reference as run in the build container (numpy's
OpenBLAS there).  The reference's leaf arithmetic is whatever `np.matmul`
does on the machine it runs on (multiply.py:255), and a different BLAS build
may order its FMAs differently, so on the GPU box the leaf stage is restated
with the box's own `np.matmul` -- batched leaf products of the retained
triples (multiply.py:224-257) merged over the inner index in aligned binary
intervals, first + second (multiply.py:119-141) -- and the CUDA product is
held to the contract bar against it: 1e-12 relative Frobenius per C block and
over the whole product.  Bit equality is reported, not required (it holds
when the host's BLAS accumulates each element as one sequential FMA chain).
"""

import numpy as np
import pytest

import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import workloads

pytestmark = pytest.mark.gpu


def _merge_tree(blocks, ks, depth):
    """Sum of one C block's leaf products over k in the reference's order:
    level by level, slots 2m and 2m+1 merge (first + second) when both are
    present, a lone slot passes through untouched."""
    cur = {int(k): blk for k, blk in zip(ks, blocks)}
    for _ in range(depth):
        nxt = {}
        for k in sorted(cur):
            if k & 1 and (k - 1) in cur:
                continue  # taken as its left neighbour's partner
            v = cur[k]
            if not k & 1 and (k + 1) in cur:
                v = v + cur[k + 1]
            nxt[k >> 1] = v
        cur = nxt
    assert len(cur) == 1
    return next(iter(cur.values()))


def _host_product(a_pad, b_pad, leaf, triples, depth, dtype):
    """{(i, j): block} from the host's np.matmul over the retained triples."""
    nb = a_pad.shape[0] // leaf
    ab = a_pad.reshape(nb, leaf, nb, leaf).swapaxes(1, 2)
    bb = b_pad.reshape(nb, leaf, nb, leaf).swapaxes(1, 2)
    order = np.lexsort((triples[:, 2], triples[:, 1], triples[:, 0]))
    t = triples[order]
    out = {}
    grp = t[:, 0].astype(np.int64) * nb + t[:, 1]
    cuts = np.flatnonzero(np.diff(grp)) + 1
    for s, e in zip(np.r_[0, cuts], np.r_[cuts, len(t)]):
        i, j = int(t[s, 0]), int(t[s, 1])
        ks = t[s:e, 2]
        prod = np.matmul(ab[i, ks].astype(dtype, copy=False), bb[ks, j].astype(dtype, copy=False))
        out[(i, j)] = _merge_tree(prod, ks, depth)
    return out


def _pad(d, leaf, depth, dtype):
    N = leaf << depth
    p = np.zeros((N, N), dtype)
    p[:d.shape[0], :d.shape[1]] = d
    return p


CASES = [
    # name, n, leaf, tau, dtype, make
    ("c1", 1024, 32, 1e-6, np.float64,
     lambda: workloads.make_config("c1")[:2]),
    ("c2_n2048", 2048, 64, 1e-8, np.float64,
     lambda: (lambda a: (a, a))(workloads.exponential_decay(2048, 0.95, 0, symmetric=True))),
    ("alg_n1000_b16", 1000, 16, 1e-7, np.float64,
     lambda: (workloads.algebraic_decay(1000, 2.0, 0), workloads.algebraic_decay(1000, 2.0, 1))),
    ("f32_n768_b32", 768, 32, 1e-5, np.float32,
     lambda: (workloads.exponential_decay(768, 0.9, 0), workloads.exponential_decay(768, 0.9, 1))),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_product_within_contract_of_host_blas(case, capsys):
    name, n, leaf, tau, dtype, make = case
    a_d, b_d = make()
    a_d = np.asarray(a_d)[:n, :n].astype(dtype)
    b_d = np.asarray(b_d)[:n, :n].astype(dtype)
    a = sp.from_dense(a_d, leaf_size=leaf, dtype=dtype)
    b = sp.from_dense(b_d, leaf_size=leaf, dtype=dtype)
    c, st, det = sp.spamm_detailed(a, b, sp.SpammConfig(tau=tau), keep_triples=True)
    depth = a.depth
    assert st.leaf_matmuls == len(det.triples) > 0
    ref = _host_product(_pad(a_d, leaf, depth, dtype), _pad(b_d, leaf, depth, dtype), leaf,
                        np.asarray(det.triples), depth, dtype)
    got = np.asarray(c._padded)
    nb = got.shape[0] // leaf
    seen = np.zeros((nb, nb), bool)
    # the bar is stated for FP64 (north_star); FP32 leaves get the same bar
    # scaled by the precision ratio
    bar = 1e-12 if dtype == np.float64 else 1e-12 * 2.0 ** 29
    num = den = 0.0
    exact = 0
    for (i, j), blk in ref.items():
        g = got[i * leaf:(i + 1) * leaf, j * leaf:(j + 1) * leaf]
        seen[i, j] = True
        d = np.linalg.norm(g.astype(np.float64) - blk.astype(np.float64))
        r = np.linalg.norm(blk.astype(np.float64))
        assert d <= bar * max(r, 1e-300), (name, i, j, d, r)
        num += d * d
        den += r * r
        exact += int(np.array_equal(g, blk))
    assert np.sqrt(num) <= bar * np.sqrt(den)
    # blocks no retained triple writes stay zero
    gz = got.reshape(nb, leaf, nb, leaf).swapaxes(1, 2)[~seen]
    assert not gz.any()
    with capsys.disabled():
        print(f"\n[host-blas] {name}: {exact}/{len(ref)} C blocks bit-equal to this host's "
              f"np.matmul merge, rel. Frobenius {np.sqrt(num / max(den, 1e-300)):.3e}")
