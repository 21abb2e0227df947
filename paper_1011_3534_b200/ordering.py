"""Morton (Z-order) keys of product-space boxes (ordering.py:24-75 of the reference).

Only the box half of the reference's ``ordering`` module is part of this
package: the i-major bit interleave that orders box logs, its ``MortonKey``
wrapper, and the key-range splitter.  The Hilbert atom ordering
(``order_atoms``, ``apply_ordering``, permutation files) is pre-processing
outside the multiply's path (out of scope).

The interleave convention is fixed by the reference: bit b of i lands at
3b + 2, of j at 3b + 1, of k at 3b.  ``write_box_log`` sorts by it on the
device (csrc/boxes.cu); the helpers here are the host-side API.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def _interleave3(i, j, k):
    """Interleave the bits of three non-negative ints, i-major (ordering.py:24-34)."""
    i, j, k = int(i), int(j), int(k)
    if i < 0 or j < 0 or k < 0:
        raise ValueError("coordinates must be non-negative")
    key = 0
    shift = 0
    while i | j | k:
        key |= (((i & 1) << 2) | ((j & 1) << 1) | (k & 1)) << shift
        i >>= 1
        j >>= 1
        k >>= 1
        shift += 3
    return key


@dataclass(frozen=True)
class MortonKey:
    """Z-order key of a product-space cuboid at a given tier (ordering.py:37-44)."""

    key: int
    tier: int


def morton_key(box, padded_dim):
    """Morton key of a pruned box in cell units of its own tier
    (ordering.py:47-55); ValueError when edge != padded_dim >> tier."""
    edge = padded_dim >> box.tier
    if edge != box.edge:
        raise ValueError(
            f"box edge {box.edge} inconsistent with tier {box.tier} "
            f"for padded_dim {padded_dim}")
    return MortonKey(_interleave3(box.i_lo // edge, box.j_lo // edge, box.k_lo // edge),
                     box.tier)


def split_key_ranges(keys, parts):
    """Split a sorted key list into ``parts`` contiguous half-open index
    ranges whose sizes differ by at most one, larger ones first
    (ordering.py:57-75)."""
    if parts < 1:
        raise ValueError(f"parts must be >= 1, got {parts}")
    keys = np.asarray(keys)
    if keys.size > 1 and bool(np.any(keys[1:] < keys[:-1])):
        raise ValueError("keys must be sorted ascending")
    base, extra = divmod(keys.size, parts)
    bounds = np.concatenate(([0], np.cumsum([base + (p < extra) for p in range(parts)])))
    return [(int(bounds[p]), int(bounds[p + 1])) for p in range(parts)]


__all__ = ["MortonKey", "morton_key", "split_key_ranges"]
