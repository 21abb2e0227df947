"""The sparse approximate matrix multiply on B200 (drop-in for ``spamm.multiply``).

``spamm(a, b, config)`` keeps the reference's signature, return value and
exceptions (multiply.py:144-221); the work runs in the CUDA library:

* K2 level-synchronous culling (csrc/traverse.cu) -- the retained leaf-triple
  set, the pruned boxes and every ProductStats integer are identical to the
  reference's, and ``omitted_budget`` is summed with numpy's pairwise order;
* K3 leaf products on the FP64 tensor-core path (csrc/leaf.cu) merged in the
  reference's binary-interval order, so C is bit-identical to the
  reference's on the same BLAS ordering;
* K1 on the product for C's norm pyramid (csrc/tree.cu).

Reference: arxiv/paper_1011_3534, pkg/src/spamm/multiply.py.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib
from .quadtree import QuadTreeMatrix, _require_conformable, _wrap, node_norm


@dataclass(frozen=True)
class SpammConfig:
    """Knobs for one multiply (multiply.py:43-74).

    ``deterministic`` is accepted for interface parity: the GPU path always
    uses the reference's fixed merge order, so results are bit-reproducible
    either way.
    """

    tau: float = 0.0
    collect_boxes: bool = False
    count_stats: bool = True
    deterministic: bool = True
    tier_tau_decay: bool = False

    def __post_init__(self):
        if not math.isfinite(self.tau) or self.tau < 0:
            raise ValueError(f"tau must be finite and >= 0, got {self.tau}")


@dataclass(frozen=True)
class PrunedBox:
    """A tau-pruned cuboid [i_lo, i_lo+edge) x [j_lo, ..) x [k_lo, ..) of the
    padded index cube, edge = padded_dim / 2**tier (multiply.py:77-90)."""

    i_lo: int
    j_lo: int
    k_lo: int
    edge: int
    tier: int


@dataclass
class ProductStats:
    """Work and truncation accounting for one multiply (multiply.py:93-116)."""

    leaf_matmuls: int = 0
    pruned_calls: int = 0
    omitted_budget: float = 0.0
    max_depth_reached: int = 0
    boxes: list | None = None
    pruned_volume: int = 0
    empty_skip_volume: int = 0

    def covered_volume(self, leaf_size):
        """Visited leaf cells + pruned boxes + Empty skips (== padded_dim**3)."""
        return (self.leaf_matmuls * leaf_size ** 3
                + self.pruned_volume + self.empty_skip_volume)


@dataclass
class MultiplyDetail:
    """Extra artefacts of one device multiply (not part of the reference API)."""

    triples: np.ndarray | None = None       # (m, 3) int32 retained (i, j, k), sorted
    tier_candidates: list = field(default_factory=list)
    tier_survivors: list = field(default_factory=list)
    tier_pruned: list = field(default_factory=list)
    n_groups: int = 0
    ms_cull: float = 0.0
    ms_leaf: float = 0.0
    ms_ctree: float = 0.0
    ms_total: float = 0.0
    ms_gemm: float = 0.0
    kernel_launches: int = 0
    traverse_phase_us: list = field(default_factory=list)
    pruned: np.ndarray | None = None        # (p, 4) int32 (tier, i, j, k), keep_pruned
    pruned_np: np.ndarray | None = None     # (p,) their norm products, reference order
    halo_bytes: int = 0                     # operand bytes fetched (distributed multiply)
    need_blocks: np.ndarray | None = None   # (nb*nb,) bool: B block (k, j) read at [k*nb+j]


def _flags(config, keep_triples, traversal="auto", traverse_only=False, keep_pruned=False,
           need_blocks=False):
    if traversal not in ("auto", "tiered"):
        raise ValueError(f"traversal must be 'auto' or 'tiered', got {traversal!r}")
    f = _lib.TIERED_TRAVERSAL if traversal == "tiered" else 0
    if traverse_only:
        f |= _lib.TRAVERSE_ONLY
    if keep_pruned:
        f |= _lib.KEEP_PRUNED
    if need_blocks:
        f |= _lib.NEED_BLOCKS
    if config.collect_boxes:
        f |= _lib.COLLECT_BOXES
    if config.count_stats:
        f |= _lib.COUNT_STATS
    if config.tier_tau_decay:
        f |= _lib.TIER_TAU_DECAY
    if keep_triples:
        f |= _lib.KEEP_TRIPLES
    return f


def spamm_detailed(a, b, config=None, keep_triples=False, rows=None, traversal="auto",
                   traverse_only=False, keep_pruned=False, need_blocks=False):
    """spamm() plus a MultiplyDetail (retained triples, per-tier counts,
    device timings).  ``rows=(lo, hi)`` restricts the product to C leaf block
    rows [lo, hi) -- the shard of one rank in the multi-GPU layout.
    ``traversal="tiered"`` forces the breadth-first tier kernel even where
    the dense single-pass kernel applies (depth <= 6); results are identical.
    ``traverse_only``: the traversal alone (no product; C is None) -- the
    multi-GPU plan.  ``keep_pruned``: the pruned calls and their norm
    products in reference order (detail.pruned / pruned_np).  ``need_blocks``:
    the B blocks the retained triples read (detail.need_blocks), formed on
    the device -- the multi-GPU plan without the triples' device->host copy."""
    _require_conformable(a, b)
    if config is None:
        config = SpammConfig()
    L = _lib.load()
    c = ctypes.c_void_p()
    prod = ctypes.c_void_p()
    st = _lib.Stats()
    flags = _flags(config, keep_triples, traversal, traverse_only, keep_pruned, need_blocks)
    if rows is None:
        _lib.check(L.spamm_multiply(a._handle, b._handle, float(config.tau), flags,
                                    ctypes.byref(c), ctypes.byref(st), ctypes.byref(prod)))
    else:
        _lib.check(L.spamm_multiply_rows(a._handle, b._handle, float(config.tau), flags,
                                         int(rows[0]), int(rows[1]), ctypes.byref(c),
                                         ctypes.byref(st), ctypes.byref(prod)))
    try:
        stats = ProductStats(boxes=[] if config.collect_boxes else None)
        stats.leaf_matmuls = int(st.leaf_matmuls)
        stats.pruned_calls = int(st.pruned_calls)
        stats.omitted_budget = float(st.omitted_budget)
        stats.max_depth_reached = int(st.max_depth_reached)
        stats.pruned_volume = int(st.pruned_volume)
        stats.empty_skip_volume = int(st.empty_skip_volume)
        depth = a.depth
        detail = MultiplyDetail(tier_candidates=list(st.tier_candidates[:depth + 1]),
                                tier_survivors=list(st.tier_survivors[:depth + 1]),
                                tier_pruned=list(st.tier_pruned[:depth + 1]),
                                n_groups=int(st.n_groups), ms_cull=st.ms_cull,
                                ms_leaf=st.ms_leaf, ms_ctree=st.ms_ctree, ms_total=st.ms_total,
                                ms_gemm=st.ms_gemm, kernel_launches=int(st.kernel_launches),
                                traverse_phase_us=list(st.traverse_phase_us))
        if config.collect_boxes and st.n_boxes:
            raw = np.empty((int(st.n_boxes), 5), np.int64)
            _lib.check(L.spamm_product_boxes(prod, raw.ctypes.data, int(st.n_boxes)))
            stats.boxes = [PrunedBox(int(x), int(y), int(z), int(e), int(t))
                           for x, y, z, e, t in raw.tolist()]
        if keep_triples:
            trip = np.empty((int(st.n_triples), 3), np.int32)
            if st.n_triples:
                _lib.check(L.spamm_product_triples(prod, trip.ctypes.data, int(st.n_triples)))
            detail.triples = trip
        if keep_pruned:
            m = int(L.spamm_product_pruned_count(prod))
            detail.pruned = np.empty((m, 4), np.int32)
            detail.pruned_np = np.empty(m, np.float64)
            if m:
                _lib.check(L.spamm_product_pruned(prod, detail.pruned.ctypes.data,
                                                  detail.pruned_np.ctypes.data, m))
        if need_blocks:
            nb = a.block_grid
            words = np.empty((nb * nb + 31) // 32, np.uint32)
            _lib.check(L.spamm_product_need_blocks(prod, words.ctypes.data, words.size))
            detail.need_blocks = np.unpackbits(words.view(np.uint8), bitorder="little")[:nb * nb] \
                .astype(bool)
    finally:
        if prod.value:
            L.spamm_product_free(prod)
    return (_wrap(c.value) if c.value else None), stats, detail


def spamm(a, b, config=None):
    """Multiply two device quadtrees with norm-product pruning
    (multiply.py:144-221).  Returns ``(QuadTreeMatrix, ProductStats)``."""
    c, stats, _ = spamm_detailed(a, b, config)
    return c, stats


def exact_multiply(a, b):
    """The exact product, tau = 0 (multiply.py:260-263)."""
    c, _ = spamm(a, b, SpammConfig(tau=0.0, count_stats=False))
    return c


def diff_norm(x, y):
    """||X - Y||_F over the padded storage, computed on the device."""
    out = ctypes.c_double()
    _lib.check(_lib.load().spamm_tree_diff_norm(x._handle, y._handle, ctypes.byref(out)))
    return float(out.value)


def multiply_error(a, b, config):
    """(abs_err, omitted_budget) of the truncated product against the exact
    one (multiply.py:266-278); the difference norm runs on the GPU."""
    if config.tau > 0 and not config.count_stats:
        config = replace(config, count_stats=True)
    approx, stats = spamm(a, b, config)
    exact = exact_multiply(a, b)
    return diff_norm(approx, exact), stats.omitted_budget


def norm_submultiplicativity_check(a, b):
    """The norm bounds pruning relies on, checked on actual data
    (multiply.py:281-303): ||AB||_F <= ||A||_F ||B||_F and, at tier 1,
    ||AB||_F <= sum over quadrant pairs of child-norm products, each with
    8 ulp of slack.  The exact product runs on the GPU."""
    _require_conformable(a, b)
    c = exact_multiply(a, b)
    slack = 1.0 + 8 * float(np.finfo(a.dtype).eps)
    nc = node_norm(c)
    if nc > node_norm(a) * node_norm(b) * slack:
        return False
    if a.depth >= 1:
        an = np.sqrt(a._norm_sq[1])
        bn = np.sqrt(b._norm_sq[1])
        bound = 0.0
        for i in range(2):
            for j in range(2):
                bound += an[i, 0] * bn[0, j] + an[i, 1] * bn[1, j]
        if nc > bound * slack:
            return False
    return True


def _box_array(boxes):
    rows = [(bx.i_lo, bx.j_lo, bx.k_lo, bx.edge, bx.tier) for bx in boxes]
    return np.array(rows, dtype=np.int64).reshape(-1, 5)


def morton_order(boxes, device=None):
    """Indices of ``boxes`` in box-log order: a stable sort by the i-major
    Morton key of (i_lo, j_lo, k_lo) (multiply.py:312, ordering.py:24-34),
    computed on the GPU (csrc/boxes.cu)."""
    from .quadtree import get_device

    arr = boxes if isinstance(boxes, np.ndarray) else _box_array(boxes)
    arr = np.ascontiguousarray(arr, dtype=np.int64).reshape(-1, 5)
    order = np.empty(arr.shape[0], np.int64)
    if arr.shape[0]:
        dev = get_device() if device is None else int(device)
        _lib.check(_lib.load().spamm_boxes_morton_order(arr.ctypes.data, arr.shape[0], dev,
                                                        order.ctypes.data))
    return order


def write_box_log(boxes, path, padded_dim):
    """Write a box log (multiply.py:306-315): one ``tier i_lo j_lo k_lo edge``
    line per pruned box, boxes in Morton order of their lower corners so that
    nearby cuboids are nearby in the file.  The order is computed on the GPU."""
    arr = _box_array(boxes)
    order = morton_order(arr)
    with open(path, "w") as fh:
        if arr.shape[0]:
            np.savetxt(fh, arr[order][:, [4, 0, 1, 2, 3]], fmt="%d", delimiter=" ")


def read_box_log(path):
    """Parse a box log written by write_box_log (multiply.py:318-328)."""
    out = []
    with open(path) as fh:
        for line in fh:
            tok = line.split()
            if not tok:
                continue
            tier, i_lo, j_lo, k_lo, edge = (int(t) for t in tok)
            out.append(PrunedBox(i_lo, j_lo, k_lo, edge, tier))
    return out


__all__ = ["SpammConfig", "PrunedBox", "ProductStats", "MultiplyDetail", "spamm",
           "spamm_detailed", "exact_multiply", "multiply_error", "diff_norm", "node_norm",
           "norm_submultiplicativity_check", "write_box_log", "read_box_log", "morton_order",
           "QuadTreeMatrix"]
