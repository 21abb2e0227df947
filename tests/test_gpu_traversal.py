"""The dense single-pass traversal (depth <= 6) against the tiered
breadth-first kernel and the oracle: identical statistics, per-tier counts,
pruned boxes (reference order), budget bits, retained triples and C, over
depths 0..7, row shards, tau sweeps and tier tau decay."""

import numpy as np
import pytest

import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import distributed as spd
from oracle import oracle

pytestmark = pytest.mark.gpu


def _decay(n, seed, rate=0.9):
    rng = np.random.default_rng(seed)
    i = np.arange(n)
    a = rng.uniform(-1, 1, (n, n)) * rate ** np.abs(i[:, None] - i[None, :])
    return (a + a.T) / 2


def _same(r1, r2):
    c1, s1, d1 = r1
    c2, s2, d2 = r2
    for k in ("leaf_matmuls", "pruned_calls", "max_depth_reached", "pruned_volume",
              "empty_skip_volume"):
        assert getattr(s1, k) == getattr(s2, k), k
    assert np.float64(s1.omitted_budget).view(np.uint64) == np.float64(s2.omitted_budget).view(np.uint64)
    assert list(d1.tier_candidates) == list(d2.tier_candidates)
    assert list(d1.tier_survivors) == list(d2.tier_survivors)
    assert list(d1.tier_pruned) == list(d2.tier_pruned)
    assert np.array_equal(d1.triples, d2.triples)
    b1 = [(b.i_lo, b.j_lo, b.k_lo, b.edge, b.tier) for b in s1.boxes]
    b2 = [(b.i_lo, b.j_lo, b.k_lo, b.edge, b.tier) for b in s2.boxes]
    assert b1 == b2
    assert np.array_equal(c1._padded.view(np.uint64), c2._padded.view(np.uint64))
    assert np.array_equal(c1._pyramid()[2].view(np.uint64), c2._pyramid()[2].view(np.uint64))


CASES = [  # (n, leaf) -> depth
    (16, 16), (40, 32), (64, 16), (128, 16), (256, 16), (512, 16), (1024, 16), (1000, 8),
]


@pytest.mark.parametrize("n,leaf", CASES)
@pytest.mark.parametrize("tau", [0.0, 1e-6, 1e-3, 0.3])
def test_dense_equals_tiered(n, leaf, tau):
    a = sp.from_dense(_decay(n, n + leaf), leaf_size=leaf)
    b = sp.from_dense(_decay(n, n + leaf + 1, 0.8), leaf_size=leaf)
    cfg = sp.SpammConfig(tau=tau, collect_boxes=True)
    _same(sp.spamm_detailed(a, b, cfg, keep_triples=True),
          sp.spamm_detailed(a, b, cfg, keep_triples=True, traversal="tiered"))


@pytest.mark.parametrize("world", [2, 3, 5])
def test_dense_shards_equal_tiered(world):
    n, leaf = 1024, 16
    a = sp.from_dense(_decay(n, 7), leaf_size=leaf)
    cfg = sp.SpammConfig(tau=1e-4, collect_boxes=True, tier_tau_decay=True)
    for r in range(world):
        rows = spd.row_shard(r, world, n, leaf)
        _same(sp.spamm_detailed(a, a, cfg, keep_triples=True, rows=rows),
              sp.spamm_detailed(a, a, cfg, keep_triples=True, rows=rows, traversal="tiered"))


def test_dense_vs_oracle_with_empty_blocks():
    # zero bands: Empty skips at several tiers, empty C blocks
    n, leaf = 512, 16
    x = _decay(n, 3)
    x[64:192, :] = 0
    x[:, 300:420] = 0
    a = sp.from_dense(x, leaf_size=leaf)
    tau = 1e-5
    c, st, det = sp.spamm_detailed(a, a, sp.SpammConfig(tau=tau, collect_boxes=True),
                                   keep_triples=True)
    pa = oracle.pad(x, leaf)
    na, oa = oracle.build_pyramid(pa, leaf)
    N = pa.shape[0]
    ost, trip, oboxes, otiers = oracle.cull(na, oa, na, oa, oracle.depth_for(N, leaf), N, tau,
                                      collect_boxes=True)
    assert st.leaf_matmuls == ost["leaf_matmuls"]
    assert st.pruned_calls == ost["pruned_calls"]
    assert st.empty_skip_volume == ost["empty_skip_volume"]
    assert st.omitted_budget == ost["omitted_budget"]
    assert np.array_equal(det.triples, np.asarray(trip, np.int32).reshape(-1, 3))
    boxes = np.array([[b.i_lo, b.j_lo, b.k_lo, b.edge, b.tier] for b in st.boxes],
                     np.int64).reshape(-1, 5)
    assert np.array_equal(boxes, oboxes)
    assert list(det.tier_candidates) == otiers["candidates"]
    assert list(det.tier_survivors) == otiers["survivors"]
    cref = oracle.leaf_stage(pa, pa, leaf, trip)
    assert np.array_equal(c._padded.view(np.uint64), cref.view(np.uint64))


def test_repeated_calls_leave_state_clean():
    # alternating depths / traversal kernels must not leak state between calls
    # (4096 at leaf 16 is depth 8: tiered traversal, separate pyramid kernel)
    mats = [(sp.from_dense(_decay(n, n), leaf_size=16), n) for n in (1024, 128, 4096, 512, 16, 1024)]
    ref = {}
    for rep in range(3):
        for a, n in mats:
            for trav in ("auto", "tiered"):
                c, st, d = sp.spamm_detailed(a, a, sp.SpammConfig(tau=1e-5), keep_triples=True,
                                             traversal=trav)
                key = n
                sig = (st.leaf_matmuls, st.pruned_calls, st.omitted_budget, d.triples.tobytes(),
                       c._padded.tobytes())
                if key in ref:
                    assert ref[key] == sig, (n, trav, rep)
                else:
                    ref[key] = sig
