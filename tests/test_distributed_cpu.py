"""Multi-process (world_size 2, gloo, CPU) coverage of the sharded layout:
each rank owns a contiguous range of C block rows (paper_1011_3534_b200.
distributed.row_shard), traverses only the triples touching it, and the
ranks exchange stats and C rows with collectives.  The oracle stands in for
the per-rank GPU kernel; the reduction/gather logic is the production code
path of paper_1011_3534_b200.distributed."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_1011_3534_b200 import distributed as spd
        from paper_1011_3534_b200 import workloads

        a, b, leaf, taus = workloads.make_config("c1")
        pa, pb = oracle.pad(a, leaf), oracle.pad(b, leaf)
        N = pa.shape[0]
        depth = oracle.depth_for(N, leaf)
        na, oa = oracle.build_pyramid(pa, leaf)
        nb_, ob = oracle.build_pyramid(pb, leaf)
        lo, hi = spd.row_shard(rank, world, a.shape[0], leaf)
        st, trip, boxes, _ = oracle.cull(na, oa, nb_, ob, depth, N, taus[0], rows=(lo, hi))
        c_local = oracle.leaf_stage(pa, pb, leaf, trip)
        stats = spd.reduce_stats(st, group=None)
        rows = c_local[lo * leaf:hi * leaf]
        full_c = spd.gather_rows(torch.from_numpy(np.ascontiguousarray(rows)), world)
        if rank == 0:
            np.save(os.path.join(out_dir, "c.npy"), full_c.numpy())
            np.save(os.path.join(out_dir, "stats.npy"),
                    np.array([stats["leaf_matmuls"], stats["pruned_calls"], stats["pruned_volume"],
                              stats["empty_skip_volume"], stats["max_depth_reached"]]))
            np.save(os.path.join(out_dir, "budget.npy"), np.array([stats["omitted_budget"]]))
    finally:
        dist.destroy_process_group()


def test_two_rank_sharded_multiply(tmp_path):
    from oracle import oracle
    from paper_1011_3534_b200 import workloads

    port = _free_port()
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, start_method="spawn")
    a, b, leaf, taus = workloads.make_config("c1")
    ref = oracle.spamm(a, b, leaf, taus[0])
    got_c = np.load(tmp_path / "c.npy")
    assert np.array_equal(got_c.view(np.uint64), ref["c_padded"].view(np.uint64))
    s = np.load(tmp_path / "stats.npy")
    r = ref["stats"]
    assert list(s) == [r["leaf_matmuls"], r["pruned_calls"], r["pruned_volume"],
                       r["empty_skip_volume"], r["max_depth_reached"]]
    budget = float(np.load(tmp_path / "budget.npy")[0])
    assert abs(budget - r["omitted_budget"]) <= 1e-12 * r["omitted_budget"]


def test_row_shard_partition():
    from paper_1011_3534_b200 import distributed as spd
    for n, leaf in ((1024, 32), (4096, 64), (1000, 4), (5, 4)):
        nb = spd.padded_blocks(n, leaf)
        for world in (1, 2, 3, 4, 8):
            spans = [spd.row_shard(r, world, n, leaf) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nb
            assert all(x[1] == y[0] for x, y in zip(spans, spans[1:]))


def test_sweep_plan_partitions_every_row_of_every_multiply_once():
    """distributed.sweep_plan: every (multiply, C block row) lands on exactly
    one rank, the plan is deterministic, and the makespan never grows with
    more ranks."""
    import numpy as np
    from paper_1011_3534_b200 import distributed as spd

    rng = np.random.default_rng(0)
    n, leaf = 4096, 64
    nb = spd.padded_blocks(n, leaf)
    counts = [rng.integers(0, 400, nb).astype(float) for _ in range(4)]
    prev = None
    for world in (1, 2, 3, 4, 8, 16):
        plan, span = spd.sweep_plan(world, n, leaf, counts)
        assert len(plan) == world
        cover = [np.zeros(nb, int) for _ in counts]
        for pieces in plan:
            for m, (lo, hi) in pieces:
                cover[m][lo:hi] += 1
        assert all((c == 1).all() for c in cover)
        assert spd.sweep_plan(world, n, leaf, counts) == (plan, span)
        if prev is not None:
            assert span <= prev + 1e-6
        prev = span


def test_row_shard_every_rank_nonempty_when_rows_suffice():
    """no rank gets an empty range while there are at least as
    many block rows as ranks -- with or without (skewed) weights; with fewer
    rows the trailing ranks get empty ranges, still covering every row once."""
    from paper_1011_3534_b200 import distributed as spd

    rng = np.random.default_rng(1)
    for n, leaf in ((1024, 32), (5, 4), (40, 4), (64, 8)):
        nb = spd.padded_blocks(n, leaf)
        for world in (1, 2, 3, 4, 8):
            for w in (None, rng.random(nb), np.r_[1.0, np.zeros(nb - 1)], np.r_[np.zeros(nb - 1), 1.0]):
                spans = [spd.row_shard(r, world, n, leaf, w) for r in range(world)]
                assert spans[0][0] == 0 and spans[-1][1] == nb
                assert all(x[1] == y[0] for x, y in zip(spans, spans[1:]))
                assert all(hi >= lo for lo, hi in spans)
                if nb >= world:
                    assert all(hi > lo for lo, hi in spans), (n, leaf, world, spans)


def _budget_worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_1011_3534_b200 import distributed as spd
        from paper_1011_3534_b200 import workloads

        a, _, leaf, taus = workloads.make_config("c2")
        pa = oracle.pad(a, leaf)
        N = pa.shape[0]
        depth = oracle.depth_for(N, leaf)
        na, oa = oracle.build_pyramid(pa, leaf)
        comm = spd.Comm()
        lo, hi = spd.row_shard(rank, world, a.shape[0], leaf)
        st, _, boxes, tiers = oracle.cull(na, oa, na, oa, depth, N, taus[2], rows=(lo, hi))
        # this rank's pruned calls as (tier, i, j, k) + norm product, gathered
        tijk = np.stack([boxes[:, 4], boxes[:, 0] // boxes[:, 3], boxes[:, 1] // boxes[:, 3],
                         boxes[:, 2] // boxes[:, 3]], axis=1) if len(boxes) else np.zeros((0, 4))
        parts_t = comm.all_gather_var(torch.from_numpy(np.ascontiguousarray(tijk, np.int64)))
        parts_v = comm.all_gather_var(torch.from_numpy(np.ascontiguousarray(tiers["box_np"])))
        tij, _, budget = spd.merge_pruned([(x.numpy(), y.numpy()) for x, y in zip(parts_t, parts_v)])
        bands = comm.bands(lo, hi)
        if rank == 0:
            np.save(os.path.join(out_dir, "merged.npy"), tij)
            np.save(os.path.join(out_dir, "budget.npy"), np.array([budget]))
            np.save(os.path.join(out_dir, "bands.npy"), np.array(bands))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_budget_is_bit_identical(tmp_path, world):
    """Per-rank pruned calls (each counted once, by the rank owning its first
    row), merged by distributed.merge_pruned into tier-major Morton order and
    pairwise-summed per tier, reproduce the single-process budget bit for bit
    and the boxes in reference order (c2 at tau = 1e-8, gloo)."""
    from oracle import oracle
    from paper_1011_3534_b200 import workloads

    port = _free_port()
    mp.start_processes(_budget_worker, args=(world, port, str(tmp_path)), nprocs=world,
                       start_method="spawn")
    a, _, leaf, taus = workloads.make_config("c2")
    ref = oracle.spamm(a, a, leaf, taus[2])
    budget = float(np.load(tmp_path / "budget.npy")[0])
    assert budget == ref["stats"]["omitted_budget"]
    b = ref["boxes"]
    want = np.stack([b[:, 4], b[:, 0] // b[:, 3], b[:, 1] // b[:, 3], b[:, 2] // b[:, 3]], axis=1)
    assert np.array_equal(np.load(tmp_path / "merged.npy"), want)
    bands = np.load(tmp_path / "bands.npy")
    assert bands[0][0] == 0 and bands[-1][1] == 64


def test_morton_keys_match_bitwise_interleave():
    """distributed.morton_keys (magic-number spreads) equals the i-major
    bit-by-bit interleave of (i, j, k) -- the candidate order inside a tier
    (multiply.py:35-37) the merged pruned list follows."""
    from paper_1011_3534_b200 import distributed as spd

    rng = np.random.default_rng(0)
    t = np.c_[rng.integers(0, 12, 4000), rng.integers(0, 2 ** 21, (4000, 3))]
    want = []
    for _, i, j, k in t.tolist():
        key = 0
        for bit in range(21):
            key |= ((i >> bit) & 1) << (3 * bit + 2)
            key |= ((j >> bit) & 1) << (3 * bit + 1)
            key |= ((k >> bit) & 1) << (3 * bit)
        want.append(key)
    assert np.array_equal(spd.morton_keys(t), np.array(want, dtype=np.uint64))
