"""Multi-GPU partitioning of the SpAMM output block space.

One process per GPU (torch.distributed; NCCL on B200s, gloo for the CPU
tests).  Rank r owns the C leaf block rows [lo_r, hi_r) (``row_shard``):

* every rank holds the operand trees (built from its row band and
  all-gathered over NVLink with ``allgather_tree``, or built locally);
* each rank runs the traversal restricted to triples whose rows touch its
  band and counts every pruned / skipped call on the rank owning the call's
  first row (``spamm_multiply_rows`` in the C ABI), so integer statistics
  sum exactly to the single-GPU ones and the retained triples partition;
* C's row bands are all-gathered (no reduction over k crosses GPUs, so the
  result is bit-identical to the single-GPU product) and its pyramid is
  rebuilt on every rank.

The reference is single-process; this module is the
B200 scale-out of its spamm() call.
"""

from __future__ import annotations

import ctypes

import numpy as np


def padded_blocks(n, leaf):
    """Leaf blocks per side of the padded matrix (quadtree.py:245-247)."""
    d = 0
    while leaf << d < n:
        d += 1
    return 1 << d


def row_shard(rank, world, n, leaf, weights=None):
    """Contiguous C block-row range of `rank`.

    Without `weights` the ranges are near-equal; with per-block-row work
    estimates (e.g. retained triples per row) they are balanced greedily by
    cumulative weight, still contiguous and covering every row once."""
    nb = padded_blocks(n, leaf)
    if weights is None:
        return (rank * nb // world, (rank + 1) * nb // world)
    w = np.asarray(weights, dtype=np.float64)
    assert w.shape == (nb,)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world)))
    cuts.append(nb)
    for r in range(1, world + 1):  # strictly increasing, every rank >= 1 row when possible
        cuts[r] = max(cuts[r], min(cuts[r - 1] + 1, nb))
    return (cuts[rank], cuts[rank + 1])


def sweep_plan(world, n, leaf, row_counts, fixed_cost=2800.0, max_split=None):
    """Partition a set of independent multiplies (e.g. a tau sweep on the same
    operands) over `world` ranks: each multiply may be split into contiguous C
    block-row shards, and the pieces are assigned to ranks (longest first).

    `row_counts[m]` are multiply m's retained triples per C block row (its
    work); a piece costs `fixed_cost` (the per-call traversal / C-tree
    overhead, in triple units: ~60 us / ~0.021 us per 64^3 triple on a B200)
    plus its rows' triples.  Shard counts are grown greedily on the multiply
    whose pieces are the most expensive while that lowers the makespan.
    Deterministic: every rank computes the same plan.

    Returns (plan, makespan): plan[r] = [(m, (row_lo, row_hi)), ...]."""
    nb = padded_blocks(n, leaf)
    counts = [np.asarray(c, dtype=np.float64) for c in row_counts]
    assert all(c.shape == (nb,) for c in counts)
    M = len(counts)
    max_split = max_split or world

    def build(splits):
        pieces = []
        for m in range(M):
            for r in range(splits[m]):
                lo, hi = row_shard(r, splits[m], n, leaf, counts[m] + 1e-9)
                if hi > lo:
                    pieces.append((fixed_cost + counts[m][lo:hi].sum(), m, (lo, hi)))
        pieces.sort(key=lambda x: (-x[0], x[1], x[2]))
        load = [0.0] * world
        plan = [[] for _ in range(world)]
        for cost, m, rows in pieces:
            r = min(range(world), key=lambda q: (load[q], q))
            load[r] += cost
            plan[r].append((m, rows))
        for p in plan:
            p.sort()
        return plan, max(load)

    splits = [1] * M
    best_plan, best = build(splits)
    while True:
        cand = [m for m in range(M) if splits[m] < max_split]
        if not cand:
            break
        # split the multiply whose pieces are the most expensive
        m = max(cand, key=lambda q: (counts[q].sum() / splits[q], -q))
        splits = list(splits)
        splits[m] += 1
        plan, span = build(splits)
        if span < best - 1e-9:
            best_plan, best = plan, span
        elif sum(splits) > world:  # more pieces than ranks and no gain: done
            break
    return best_plan, best


_INT_KEYS = ("leaf_matmuls", "pruned_calls", "pruned_volume", "empty_skip_volume")


def reduce_stats(stats, group=None):
    """Sum per-rank ProductStats (or dicts) over the group.

    Integers are summed exactly; max_depth_reached is the max; the budgets are
    all-gathered and added in rank order on every rank, so the result is
    deterministic and identical everywhere."""
    import torch
    import torch.distributed as dist

    get = (lambda k: stats[k]) if isinstance(stats, dict) else (lambda k: getattr(stats, k))
    world = dist.get_world_size(group)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    ints = torch.tensor([get(k) for k in _INT_KEYS] + [get("max_depth_reached")],
                        dtype=torch.int64, device=dev)
    flo = torch.tensor([get("omitted_budget")], dtype=torch.float64, device=dev)
    all_i = [torch.empty_like(ints) for _ in range(world)]
    all_f = [torch.empty_like(flo) for _ in range(world)]
    dist.all_gather(all_i, ints, group=group)
    dist.all_gather(all_f, flo, group=group)
    out = {k: int(sum(int(t[q]) for t in all_i)) for q, k in enumerate(_INT_KEYS)}
    out["max_depth_reached"] = int(max(int(t[len(_INT_KEYS)]) for t in all_i))
    budget = 0.0
    for t in all_f:  # fixed rank order
        budget += float(t[0])
    out["omitted_budget"] = budget
    return out


def gather_rows(local_rows, world, group=None):
    """All-gather row bands (possibly of different heights) into one array,
    rank order = row order."""
    import torch
    import torch.distributed as dist

    h = torch.tensor([local_rows.shape[0]], dtype=torch.int64, device=local_rows.device)
    hs = [torch.empty_like(h) for _ in range(world)]
    dist.all_gather(hs, h, group=group)
    heights = [int(x) for x in hs]
    hmax = max(heights)
    if local_rows.shape[0] < hmax:
        pad = torch.zeros((hmax - local_rows.shape[0],) + tuple(local_rows.shape[1:]),
                          dtype=local_rows.dtype, device=local_rows.device)
        local_rows = torch.cat([local_rows, pad])
    bufs = [torch.empty_like(local_rows) for _ in range(world)]
    dist.all_gather(bufs, local_rows.contiguous(), group=group)
    return torch.cat([b[:hh] for b, hh in zip(bufs, heights)])


class DeviceArray:
    """A borrowed view of device memory exposing __cuda_array_interface__,
    so torch (NCCL collectives) can operate on a tree's storage in place."""

    def __init__(self, ptr, shape, dtype):
        self.ptr, self.shape, self.dtype = int(ptr), tuple(shape), np.dtype(dtype)

    @property
    def __cuda_array_interface__(self):
        return {"shape": self.shape, "typestr": self.dtype.str, "data": (self.ptr, False),
                "version": 3, "strides": None}


def tree_storage(tree):
    """torch view of a tree's padded N x N device storage (borrowed)."""
    import torch
    from . import _lib

    p = ctypes.c_void_p()
    _lib.check(_lib.load().spamm_tree_device_ptrs(tree._handle, ctypes.byref(p), None, None))
    return torch.as_tensor(DeviceArray(p.value, (tree.padded_dim, tree.padded_dim), tree.dtype),
                           device=f"cuda:{tree.device}")


def tree_from_padded(padded, n, leaf, device=None):
    """Adopt a padded N x N torch CUDA tensor as a tree (copied; pyramid rebuilt)."""
    from . import _lib
    from .quadtree import _wrap

    assert padded.is_cuda and padded.is_contiguous()
    from .quadtree import _sync_torch

    _sync_torch()  # torch's collectives/kernels that filled `padded` come first
    code = _lib.DTYPE_F64 if padded.dtype == __import__("torch").float64 else _lib.DTYPE_F32
    h = ctypes.c_void_p()
    dev = padded.device.index if device is None else device
    _lib.check(_lib.load().spamm_tree_from_padded_device(
        ctypes.c_void_p(padded.data_ptr()), int(n), int(padded.shape[0]), int(leaf), code, dev,
        ctypes.byref(h)))
    return _wrap(h.value)


def allgather_tree(local_rows, n, leaf, group=None):
    """Build the same tree on every rank from row bands of the padded matrix.

    `local_rows` is this rank's (h_r x N) band of the zero-padded input as a
    CUDA tensor (rank order = row order); the bands are all-gathered over
    NCCL / NVLink and every rank builds the norm pyramid locally."""
    import torch.distributed as dist

    full = gather_rows(local_rows, dist.get_world_size(group), group)
    return tree_from_padded(full.contiguous(), n, leaf)


def spamm_sharded(a, b, config=None, group=None, weights=None):
    """spamm() with the C block rows partitioned over the process group.

    Returns (C, stats_dict, detail) on every rank; C is the full product
    (bit-identical to the single-GPU result), stats are the exact sums."""
    import torch.distributed as dist
    from .multiply import spamm_detailed

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = row_shard(rank, world, a.logical_dim, a.leaf_size, weights)
    c_local, st, det = spamm_detailed(a, b, config, rows=(lo, hi))
    leaf = a.leaf_size
    rows = tree_storage(c_local)[lo * leaf:hi * leaf]
    c = allgather_tree(rows, a.logical_dim, leaf, group)
    return c, reduce_stats(st, group), det
