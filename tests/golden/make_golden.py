"""Generate the golden fixtures by running the REAL reference package.

Run in the build container (the only place /root/reference exists):

    SPAMM_REF=/root/reference/pkg/src python tests/golden/make_golden.py

For every case it imports the reference `spamm` package, builds trees with
`from_dense`, runs `spamm(A, B, SpammConfig(...))` and records:

* the norm / occupancy pyramids of A, B and C (`_norm_sq`, `_occupied`),
* the retained leaf triples, captured from the reference's own
  `_leaf_stage` (multiply.py:224) by wrapping it -- the reference does not
  otherwise expose them,
* ProductStats (integers exact, budget as the exact float) and the pruned
  boxes in the reference's order,
* C (full padded array for small cases; for large ones a 64-bit hash of
  every nonzero block -- ``block_hash`` -- plus eight blocks as stored) and
  the SpAMM-vs-exact error ``multiply_error``.

``GOLDEN_ONLY=c1,c3_l2_tau1e-08 python tests/golden/make_golden.py``
regenerates just the named large cases and merges them into golden.json.

Inputs are regenerated from seeds at test time (numpy PCG64 is
bit-reproducible), so only the small-case inputs are stored.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.environ.get("SPAMM_REF", "/root/reference/pkg/src"))
sys.dont_write_bytecode = True

import spamm  # noqa: E402  (the reference)
import spamm.multiply as ref_multiply  # noqa: E402
from spamm import SpammConfig, from_dense, multiply_error, spamm as ref_spamm  # noqa: E402

from paper_1011_3534_b200 import workloads  # noqa: E402

_captured = []
_orig_leaf_stage = ref_multiply._leaf_stage


def _capturing_leaf_stage(a, b, out_blocks, ia, ja, ka, nb, depth, stats, counting):
    _captured.append((ia.copy(), ja.copy(), ka.copy()))
    return _orig_leaf_stage(a, b, out_blocks, ia, ja, ka, nb, depth, stats, counting)


ref_multiply._leaf_stage = _capturing_leaf_stage


def pyramid(t):
    nsq = np.concatenate([np.asarray(x, dtype=np.float64).ravel() for x in t._norm_sq])
    occ = np.concatenate([np.asarray(x, dtype=np.uint8).ravel() for x in t._occupied])
    return nsq, occ


HASH_SEED = 77


def hash_keys(leaf):
    """Odd 64-bit multipliers, one per element of a leaf block."""
    rng = np.random.default_rng(HASH_SEED)
    return rng.integers(0, 2 ** 63, size=leaf * leaf, dtype=np.uint64) * np.uint64(2) + np.uint64(1)


def block_hash(blocks):
    """h = sum_e bits(x_e) * K_e mod 2^64 per block ((m, b, b) array): any
    change of any element's bits changes h (K_e odd)."""
    m, b = blocks.shape[0], blocks.shape[1]
    bits = np.ascontiguousarray(blocks).view(np.uint32 if blocks.dtype == np.float32
                                             else np.uint64).reshape(m, b * b).astype(np.uint64)
    with np.errstate(over="ignore"):
        return (bits * hash_keys(b)[None, :]).sum(axis=1, dtype=np.uint64)


def c_block_hashes(c):
    """(leaf ids i * nb + j, hashes) of every nonzero leaf of the reference's C."""
    nz = np.argwhere(np.asarray(c._leaf_nonzero))
    nbk = c.block_grid
    ids = (nz[:, 0] * nbk + nz[:, 1]).astype(np.int64)
    out = np.empty(len(ids), np.uint64)
    for s in range(0, len(ids), 4096):
        blk = np.stack([np.asarray(c._blocks[i, j]) for i, j in nz[s:s + 4096]])
        out[s:s + 4096] = block_hash(blk)
    return ids, out


def run_case(name, ad, bd, leaf, tau, dtype=None, tier_tau_decay=False, store_inputs=False,
             store_c="full", recipe=None):
    a = from_dense(ad, leaf_size=leaf, dtype=dtype)
    b = a if bd is ad else from_dense(bd, leaf_size=leaf, dtype=dtype)
    cfg = SpammConfig(tau=tau, collect_boxes=True, tier_tau_decay=tier_tau_decay)
    _captured.clear()
    c, st = ref_spamm(a, b, cfg)
    if _captured:
        ia, ja, ka = _captured[0]
        order = np.lexsort((ka, ja, ia))
        trip = np.stack([ia[order], ja[order], ka[order]], axis=1).astype(np.int32)
    else:
        trip = np.zeros((0, 3), np.int32)
    assert len(trip) == st.leaf_matmuls, (name, len(trip), st.leaf_matmuls)
    boxes = np.array([[bx.i_lo, bx.j_lo, bx.k_lo, bx.edge, bx.tier] for bx in st.boxes],
                     dtype=np.int64).reshape(-1, 5)
    abs_err, budget = multiply_error(a, b, SpammConfig(tau=tau, tier_tau_decay=tier_tau_decay))
    na, oa = pyramid(a)
    nb_, ob = pyramid(b)
    nc, oc = pyramid(c)
    arrays = dict(nsq_a=na, occ_a=oa, nsq_b=nb_, occ_b=ob, nsq_c=nc, occ_c=oc,
                  triples=trip.astype(np.int16 if a.block_grid < 32768 else np.int32),
                  boxes=boxes)
    if store_inputs:
        arrays["a"] = np.asarray(ad)
        arrays["b"] = np.asarray(bd)
    if store_c == "full":
        arrays["c_padded"] = np.asarray(c._padded)
    else:
        # every nonzero C block pinned by a 64-bit linear hash of its bits
        # (block_hash below), plus a handful of blocks kept as stored
        ids, hashes = c_block_hashes(c)
        arrays["c_block_ids"] = ids
        arrays["c_block_hash"] = hashes
        nbk = a.block_grid
        rng = np.random.default_rng(123)
        occ_leaf = np.argwhere(np.asarray(c._leaf_nonzero))
        pick = occ_leaf[rng.choice(len(occ_leaf), size=min(8, len(occ_leaf)), replace=False)]
        arrays["c_sample_ij"] = pick.astype(np.int32)
        arrays["c_sample"] = np.stack([np.asarray(c._blocks[i, j]) for i, j in pick]) if len(pick) \
            else np.zeros((0, leaf, leaf))
        assert nbk == c.block_grid
    meta = dict(name=name, n=int(a.logical_dim), leaf=int(leaf), depth=int(a.depth),
                padded_dim=int(a.padded_dim), tau=float(tau), dtype=str(a.dtype),
                tier_tau_decay=bool(tier_tau_decay), same_operand=bool(bd is ad),
                recipe=recipe,
                stats=dict(leaf_matmuls=int(st.leaf_matmuls), pruned_calls=int(st.pruned_calls),
                           omitted_budget=float(st.omitted_budget),
                           omitted_budget_hex=float(st.omitted_budget).hex(),
                           max_depth_reached=int(st.max_depth_reached),
                           pruned_volume=int(st.pruned_volume),
                           empty_skip_volume=int(st.empty_skip_volume),
                           n_boxes=len(st.boxes)),
                abs_err=float(abs_err), budget_from_error_run=float(budget),
                norm_a=float(a.norm()), norm_b=float(b.norm()), norm_c=float(c.norm()))
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **arrays)
    return meta


def main():
    only = [x for x in os.environ.get("GOLDEN_ONLY", "").split(",") if x]
    if only:  # regenerate just these cases, keeping the others' records
        return main_only(only)
    metas = []
    rng = np.random.default_rng(20261020)
    # -- small white-box cases (inputs stored): padding, leaf sizes, zeros, -0.0, f32
    small = []
    for n, leaf, tau in [(1, 1, 0.0), (5, 4, 0.0), (13, 2, 1e-3), (33, 4, 1e-2), (64, 8, 1e-1),
                         (100, 4, 1e-4), (64, 16, 0.5), (40, 1, 1e-2)]:
        idx = np.arange(n)
        dec = np.exp(-0.7 * np.abs(idx[:, None] - idx[None, :]))
        small.append((f"small_n{n}_b{leaf}", dec * rng.standard_normal((n, n)),
                      dec * rng.standard_normal((n, n)), leaf, tau, None, False))
    z = np.zeros((24, 24)); z[:8, :8] = -0.0; z[16:, 16:] = rng.standard_normal((8, 8))
    small.append(("zeros_negzero_n24_b4", z, rng.standard_normal((24, 24)), 4, 0.0, None, False))
    small.append(("identity_n64_b4", np.eye(64), np.eye(64), 4, 0.0, None, False))
    e = np.exp(-1.0 * np.abs(np.arange(128)[:, None] - np.arange(128)[None, :]))
    small.append(("tierdecay_n128_b4", e * rng.standard_normal((128, 128)),
                  e * rng.standard_normal((128, 128)), 4, 1e-6, None, True))
    small.append(("f32_n96_b8", (e[:96, :96] * rng.standard_normal((96, 96))).astype(np.float32),
                  (e[:96, :96] * rng.standard_normal((96, 96))).astype(np.float32), 8, 1e-5,
                  np.float32, False))
    big_tau = rng.standard_normal((16, 16))
    small.append(("rootprune_n16_b4", big_tau, rng.standard_normal((16, 16)), 4, 1e3, None, False))
    for name, ad, bd, leaf, tau, dt, decay in small:
        metas.append(run_case(name, ad, bd, leaf, tau, dtype=dt, tier_tau_decay=decay,
                              store_inputs=True, store_c="full"))
        print(metas[-1]["name"], metas[-1]["stats"])

    # -- the reference's own n=512 exponential pair (test_multiply.py:158-168)
    idx = np.arange(512)
    d = np.abs(idx[:, None] - idx[None, :])
    metas.append(run_case("refpair_n512_b4", np.exp(-1.0 * d), np.exp(-2.0 * d), 4, 1e-8,
                          store_c="sample", recipe="exp(-alpha*|i-j|), alpha=1.0 / 2.0"))
    print(metas[-1]["name"], metas[-1]["stats"])

    # -- BASELINE.json configs (inputs regenerated from seeds at test time)
    a, b, leaf, taus = workloads.make_config("c1")
    metas.append(run_case("c1", a, b, leaf, taus[0], store_c="sample", recipe="workloads:c1"))
    print(metas[-1]["name"], metas[-1]["stats"])
    a, b, leaf, taus = workloads.make_config("c2")
    for tau in taus:
        metas.append(run_case(f"c2_tau{tau:.0e}", a, a, leaf, tau, store_c="sample",
                              recipe="workloads:c2"))
        print(metas[-1]["name"], metas[-1]["stats"])
    if os.environ.get("GOLDEN_LARGE", "1") == "1":
        a, b, leaf, taus = workloads.make_config("c3_l3")
        for tau in taus:
            metas.append(run_case(f"c3_l3_tau{tau:.0e}", a, b, leaf, tau, store_c="sample",
                                  recipe="workloads:c3_l3"))
            print(metas[-1]["name"], metas[-1]["stats"])
        a, b, leaf, taus = workloads.make_config("c3_l2")
        for tau in taus:
            metas.append(run_case(f"c3_l2_tau{tau:.0e}", a, b, leaf, tau, store_c="sample",
                                  recipe="workloads:c3_l2"))
            print(metas[-1]["name"], metas[-1]["stats"])
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(dict(generator="tests/golden/make_golden.py",
                       reference="arxiv/paper_1011_3534 spamm 0.1.0 (pkg/src/spamm)",
                       numpy=np.__version__, cases=metas), fh, indent=1)


def large_case(name):
    """(inputs, leaf, tau, recipe) of a seeded BASELINE-config case by name."""
    if name == "refpair_n512_b4":
        d = np.abs(np.arange(512)[:, None] - np.arange(512)[None, :])
        return np.exp(-1.0 * d), np.exp(-2.0 * d), 4, 1e-8, "exp(-alpha*|i-j|), alpha=1.0 / 2.0"
    cfg = name.split("_tau")[0]
    a, b, leaf, taus = workloads.make_config(cfg)
    tau = float(name.split("_tau")[1]) if "_tau" in name else taus[0]
    return a, (a if cfg == "c2" else b), leaf, tau, f"workloads:{cfg}"


def main_only(names):
    path = os.path.join(HERE, "golden.json")
    with open(path) as fh:
        doc = json.load(fh)
    by_name = {c["name"]: c for c in doc["cases"]}
    for name in names:
        a, b, leaf, tau, recipe = large_case(name)
        meta = run_case(name, a, b, leaf, tau, store_c="sample", recipe=recipe)
        print(meta["name"], meta["stats"], flush=True)
        if name in by_name:
            doc["cases"][[c["name"] for c in doc["cases"]].index(name)] = meta
        else:
            doc["cases"].append(meta)
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1)


if __name__ == "__main__":
    main()
