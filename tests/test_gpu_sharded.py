"""Row-sharded multiplies (the multi-GPU layout) on one B200: the C ABI's
spamm_multiply_rows shards must partition the retained triples, sum to the
unsharded statistics exactly and reproduce C's rows bit for bit; and the
torch.distributed plumbing (NCCL, world size 1) assembles the full tree."""

import os
import socket

import numpy as np
import pytest

import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import distributed as spd
from paper_1011_3534_b200 import workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 8])
def test_row_shards_partition_the_product(world):
    a_d = workloads.exponential_decay(4096, 0.95, 0, symmetric=True)
    a = sp.from_dense(a_d, leaf_size=64)
    cfg = sp.SpammConfig(tau=1e-8, collect_boxes=True)
    full_c, full_st, full_det = sp.spamm_detailed(a, a, cfg, keep_triples=True)
    tot = dict.fromkeys(["leaf_matmuls", "pruned_calls", "pruned_volume", "empty_skip_volume"], 0)
    trips, nbox, depth, budget = [], 0, 0, 0.0
    full_pad = full_c._padded
    for r in range(world):
        lo, hi = spd.row_shard(r, world, a.logical_dim, a.leaf_size)
        c, st, det = sp.spamm_detailed(a, a, cfg, keep_triples=True, rows=(lo, hi))
        for k in tot:
            tot[k] += getattr(st, k)
        depth = max(depth, st.max_depth_reached)
        budget += st.omitted_budget
        nbox += len(st.boxes)
        trips.append(det.triples)
        rows = slice(lo * 64, hi * 64)
        assert np.array_equal(c._padded[rows].view(np.uint64), full_pad[rows].view(np.uint64))
        other = np.ones(full_pad.shape[0], bool)
        other[rows] = False
        assert not c._padded[other].any()
    for k in tot:
        assert tot[k] == getattr(full_st, k), k
    assert depth == full_st.max_depth_reached
    assert abs(budget - full_st.omitted_budget) <= 1e-12 * full_st.omitted_budget
    assert nbox == len(full_st.boxes)
    assert np.array_equal(np.concatenate(trips), full_det.triples)
