"""Multi-GPU partitioning of the SpAMM output block space.

One process per GPU.  Rank r owns the C leaf block rows [lo_r, hi_r); it
traverses only the product-space triples whose rows intersect its range and
counts each pruned / skipped call on the rank owning the call's first row,
so the per-rank integer statistics sum exactly to the single-GPU ones.
"""

from __future__ import annotations


def padded_blocks(n, leaf):
    d = 0
    while leaf << d < n:
        d += 1
    return 1 << d


def row_shard(rank, world, n, leaf):
    """Contiguous, near-equal C block-row range of `rank` (leaf block units)."""
    nb = padded_blocks(n, leaf)
    return (rank * nb // world, (rank + 1) * nb // world)
