"""ctypes wrapper over oracle/_build/libspamm_oracle.so.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Functions mirror the
reference's steps: `pad` (quadtree.py:245-250), `build_pyramid`
(quadtree.py:116-151), `cull` (multiply.py:174-212), `leaf_stage`
(multiply.py:224-257) and `spamm` composing them (multiply.py:144-221).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libspamm_oracle.so")
_lib = None


class _CullResult(ctypes.Structure):
    _fields_ = [("leaf_matmuls", ctypes.c_int64), ("pruned_calls", ctypes.c_int64),
                ("pruned_volume", ctypes.c_int64), ("empty_skip_volume", ctypes.c_int64),
                ("max_depth_reached", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("omitted_budget", ctypes.c_double),
                ("n_triples", ctypes.c_int64), ("triples", ctypes.POINTER(ctypes.c_int32)),
                ("n_boxes", ctypes.c_int64), ("boxes", ctypes.POINTER(ctypes.c_int64)),
                ("tier_candidates", ctypes.c_int64 * 32),
                ("tier_survivors", ctypes.c_int64 * 32),
                ("box_np", ctypes.POINTER(ctypes.c_double))]


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i64, i32, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        L.oracle_depth.argtypes = [i64, i32]
        L.oracle_depth.restype = ctypes.c_int
        L.oracle_build_pyramid.argtypes = [vp, ctypes.c_int, i64, i32, vp, vp]
        L.oracle_pairwise_sum.argtypes = [vp, i64]
        L.oracle_pairwise_sum.restype = dp
        L.oracle_cull.argtypes = [vp, vp, vp, vp, ctypes.c_int, i64, dp, ctypes.c_int,
                                  ctypes.c_int, ctypes.c_int, ctypes.POINTER(_CullResult)]
        L.oracle_cull.restype = ctypes.c_int
        L.oracle_cull_rows.argtypes = [vp, vp, vp, vp, ctypes.c_int, i64, dp, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, i64, i64,
                                       ctypes.POINTER(_CullResult)]
        L.oracle_cull_rows.restype = ctypes.c_int
        L.oracle_leaf_stage.argtypes = [vp, vp, ctypes.c_int, i64, i32, vp, i64, vp]
        L.oracle_leaf_stage.restype = ctypes.c_int
        L.oracle_free.argtypes = [vp]
        L.oracle_leaf_norms.argtypes = [vp, ctypes.c_int, i64, i32, vp, vp]
        L.oracle_pyramid_from_leaves.argtypes = [vp, vp, ctypes.c_int]
        L.oracle_group_product.argtypes = [vp, vp, ctypes.c_int, i32, vp, i64, ctypes.c_int, vp]
        L.oracle_group_product.restype = ctypes.c_int
        _lib = L
    return _lib


def depth_for(n, leaf):
    d = 0
    while leaf << d < n:
        d += 1
    return d


def pad(dense, leaf, dtype=np.float64):
    arr = np.asarray(dense, dtype=dtype)
    n = arr.shape[0]
    big = leaf << depth_for(n, leaf)
    out = np.zeros((big, big), dtype=dtype)
    out[:n, :n] = arr
    return out


def pyramid_size(depth):
    return ((1 << (2 * (depth + 1))) - 1) // 3


def level_slices(depth):
    off = 0
    out = []
    for k in range(depth + 1):
        out.append(slice(off, off + (1 << (2 * k))))
        off += 1 << (2 * k)
    return out


def build_pyramid(padded, leaf):
    """Canonicalises `padded` in place; returns (nsq, occ) concatenated levels."""
    assert padded.flags.c_contiguous
    N = padded.shape[0]
    depth = depth_for(N, leaf)
    nsq = np.zeros(pyramid_size(depth), np.float64)
    occ = np.zeros(pyramid_size(depth), np.uint8)
    dt = 0 if padded.dtype == np.float64 else 1
    lib().oracle_build_pyramid(padded.ctypes.data, dt, N, leaf, nsq.ctypes.data, occ.ctypes.data)
    return nsq, occ


def cull(nsq_a, occ_a, nsq_b, occ_b, depth, N, tau, tier_tau_decay=False, count_stats=True,
         collect_boxes=True, rows=None):
    """Tier traversal; ``rows=(lo, hi)`` restricts it to a C block-row shard."""
    r = _CullResult()
    L = lib()
    lo, hi = (0, 1 << depth) if rows is None else rows
    rc = L.oracle_cull_rows(nsq_a.ctypes.data, occ_a.ctypes.data, nsq_b.ctypes.data,
                            occ_b.ctypes.data, depth, N, float(tau), int(tier_tau_decay),
                            int(count_stats), int(collect_boxes), int(lo), int(hi),
                            ctypes.byref(r))
    if rc != 0:
        raise MemoryError("oracle_cull failed")
    trip = np.ctypeslib.as_array(r.triples, shape=(r.n_triples, 3)).copy() if r.n_triples \
        else np.zeros((0, 3), np.int32)
    boxes = np.ctypeslib.as_array(r.boxes, shape=(r.n_boxes, 5)).copy() if r.n_boxes \
        else np.zeros((0, 5), np.int64)
    box_np = np.ctypeslib.as_array(r.box_np, shape=(r.n_boxes,)).copy() if r.n_boxes \
        else np.zeros(0)
    L.oracle_free(ctypes.cast(r.triples, ctypes.c_void_p))
    L.oracle_free(ctypes.cast(r.boxes, ctypes.c_void_p))
    L.oracle_free(ctypes.cast(r.box_np, ctypes.c_void_p))
    stats = dict(leaf_matmuls=r.leaf_matmuls, pruned_calls=r.pruned_calls,
                 omitted_budget=r.omitted_budget, max_depth_reached=r.max_depth_reached,
                 pruned_volume=r.pruned_volume, empty_skip_volume=r.empty_skip_volume)
    tiers = dict(candidates=list(r.tier_candidates[:depth + 1]),
                 survivors=list(r.tier_survivors[:depth + 1]), box_np=box_np)
    return stats, trip, boxes, tiers


def leaf_stage(pa, pb, leaf, triples):
    N = pa.shape[0]
    c = np.zeros_like(pa)
    t = np.ascontiguousarray(triples, dtype=np.int32)
    dt = 0 if pa.dtype == np.float64 else 1
    rc = lib().oracle_leaf_stage(pa.ctypes.data, pb.ctypes.data, dt, N, leaf, t.ctypes.data,
                                 len(t), c.ctypes.data)
    if rc != 0:
        raise MemoryError("oracle_leaf_stage failed")
    return c


def spamm(ad, bd, leaf, tau, dtype=np.float64, tier_tau_decay=False, collect_boxes=True):
    """Full oracle multiply on dense inputs; returns a dict of every artefact."""
    pa = pad(ad, leaf, dtype)
    pb = pa if bd is ad else pad(bd, leaf, dtype)
    N = pa.shape[0]
    depth = depth_for(N, leaf)
    na, oa = build_pyramid(pa, leaf)
    nb, ob = (na, oa) if pb is pa else build_pyramid(pb, leaf)
    stats, trip, boxes, tiers = cull(na, oa, nb, ob, depth, N, tau, tier_tau_decay,
                                     True, collect_boxes)
    c = leaf_stage(pa, pb, leaf, trip)
    nc, oc = build_pyramid(c, leaf)
    return dict(a_padded=pa, b_padded=pb, nsq_a=na, occ_a=oa, nsq_b=nb, occ_b=ob,
                stats=stats, triples=trip, boxes=boxes, tiers=tiers,
                c_padded=c, nsq_c=nc, occ_c=oc, depth=depth, N=N)


# ----------------------------------- pieces for trees too large to hold densely
def leaf_norms(blocks):
    """(nsq, occ) of contiguous (count, b, b) leaf blocks (quadtree.py:74-87, :126)."""
    blocks = np.ascontiguousarray(blocks)
    count, leaf = blocks.shape[0], blocks.shape[1]
    nsq = np.zeros(count, np.float64)
    occ = np.zeros(count, np.uint8)
    dt = 0 if blocks.dtype == np.float64 else 1
    if count:
        lib().oracle_leaf_norms(blocks.ctypes.data, dt, count, leaf, nsq.ctypes.data,
                                occ.ctypes.data)
    return nsq, occ


def pyramid_from_leaves(nsq_leaf, occ_leaf, depth):
    """Concatenated (nsq, occ) pyramids from the leaf level (row-major nb x nb)
    by the reference's parent sums and occupancy OR (quadtree.py:90-92, :135-138)."""
    nsq = np.zeros(pyramid_size(depth), np.float64)
    occ = np.zeros(pyramid_size(depth), np.uint8)
    lv = level_slices(depth)[depth]
    nsq[lv] = np.asarray(nsq_leaf, np.float64).ravel()
    occ[lv] = np.asarray(occ_leaf, np.uint8).ravel()
    lib().oracle_pyramid_from_leaves(nsq.ctypes.data, occ.ctypes.data, depth)
    return nsq, occ


def group_product(a_blocks, b_blocks, ks, depth):
    """One C block of _leaf_stage (multiply.py:224-257): A(i, k) B(k, j) over the
    ascending retained ks, merged in the reference's binary-interval order over
    [0, 2^depth) (multiply.py:119-141).  a_blocks / b_blocks: (len(ks), b, b)."""
    a_blocks = np.ascontiguousarray(a_blocks)
    b_blocks = np.ascontiguousarray(b_blocks, dtype=a_blocks.dtype)
    ks = np.ascontiguousarray(ks, dtype=np.int32)
    leaf = a_blocks.shape[1]
    out = np.zeros((leaf, leaf), a_blocks.dtype)
    dt = 0 if a_blocks.dtype == np.float64 else 1
    rc = lib().oracle_group_product(a_blocks.ctypes.data, b_blocks.ctypes.data, dt, leaf,
                                    ks.ctypes.data, len(ks), depth, out.ctypes.data)
    if rc != 0:
        raise MemoryError("oracle_group_product failed")
    return out
