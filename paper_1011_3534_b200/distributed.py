"""Multi-GPU partitioning of the SpAMM output block space.

One process per GPU (torch.distributed; NCCL on B200s, gloo for host-side
tests).  A matrix is distributed by C block rows: rank r holds a
:class:`ShardedTree` -- a band tree (csrc/shard.cu) with the element storage
of its block rows [lo_r, hi_r) (``row_shard``) and the WHOLE matrix's norm /
occupancy pyramid.  Nothing dense is ever all-gathered:

* **pyramids** -- each rank forms its band's leaf norms, the leaf level is
  all-gathered (9 bytes per leaf block: 9.4 MB for the whole c5 matrix) and
  every rank rebuilds the levels above in the reference's fixed order
  (quadtree.py:90-92), so all ranks hold bit-identical pyramids;
* **operands** -- a row shard of C = A B traverses from the root with the
  global pyramids (``spamm_multiply_rows``: only triples whose rows meet the
  band; each pruned / skipped call counted by the rank owning its first row),
  first in plan mode to list the B blocks its retained triples read, then
  fetches exactly the ones held by other ranks (``halo_exchange``: an
  all-to-all of block ids, then of the blocks) before running the products;
* **C** stays a band per rank: its leaf level is all-gathered for the global
  pyramid (the next multiply's operand, SP2's iterate); the elements are
  gathered only on demand (``gather_padded`` / ``gather_dense``);
* **statistics** -- integers summed exactly; the budget rebuilt bit for bit:
  the ranks' pruned calls (tier, i, j, k, norm product) are merged into the
  single-GPU order (tier-major, then the Morton order of the candidates,
  multiply.py:35-37) and summed with numpy's pairwise sum per tier
  (multiply.py:197), so every ProductStats field equals the single-GPU one.

``purify_sharded`` runs the TC2 driver (purification.py:105-227) on such
matrices: per sweep a sharded square, one fused band pass (spamm_tc2_update)
and gathered leaf levels -- densities, traces, leaf counts and energies
bit-identical to the single-GPU driver.

The reference is single-process; this module is the B200
scale-out of its spamm() call and its purification driver.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib


# ------------------------------------------------------------- partitioning
def padded_blocks(n, leaf):
    """Leaf blocks per side of the padded matrix (quadtree.py:245-247)."""
    d = 0
    while leaf << d < n:
        d += 1
    return 1 << d


def row_shard(rank, world, n, leaf, weights=None):
    """Contiguous C block-row range [lo, hi) of `rank`.

    The ranges cover every block row once, in rank order.  When there are at
    least as many block rows as ranks every range holds at least one row;
    with fewer, the trailing ranks get empty ranges (lo == hi), which every
    collective in this module still joins.  Without `weights` the ranges are
    near-equal; with per-block-row work estimates (e.g. retained triples per
    row) they are balanced by cumulative weight."""
    nb = padded_blocks(n, leaf)
    if weights is None:
        cuts = [r * nb // world for r in range(world)] + [nb]
        if nb < world:
            cuts = [min(r, nb) for r in range(world)] + [nb]
        return (cuts[rank], cuts[rank + 1])
    w = np.asarray(weights, dtype=np.float64)
    assert w.shape == (nb,)
    cum = np.concatenate([[0.0], np.cumsum(w)])
    total = cum[-1]
    cuts = [0] + [int(np.searchsorted(cum, total * r / world)) for r in range(1, world)] + [nb]
    for r in range(1, world):  # non-decreasing, and >= 1 row per rank while rows remain
        lo_bound = cuts[r - 1] + (1 if nb >= world else 0)
        hi_bound = nb - (world - r) if nb >= world else nb
        cuts[r] = min(max(cuts[r], lo_bound), max(hi_bound, lo_bound))
        cuts[r] = min(cuts[r], nb)
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


# --------------------------------------------------- budget in reference order
def morton_keys(tier_ijk):
    """i-major interleave of (i, j, k) -- a candidate's position in its tier's
    breadth-first list (children (di, dj, dk) = 000..111, multiply.py:35-37)."""
    t = np.asarray(tier_ijk, dtype=np.int64).reshape(-1, 4)

    def spread3(x):  # bit b of a 21-bit x -> bit 3b
        x = x.astype(np.uint64) & np.uint64(0x1FFFFF)
        for shift, mask in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                            (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
            x = (x | (x << np.uint64(shift))) & np.uint64(mask)
        return x

    return (spread3(t[:, 1]) << np.uint64(2)) | (spread3(t[:, 2]) << np.uint64(1)) | spread3(t[:, 3])


def merge_pruned(parts):
    """Merge per-rank pruned-call lists [(tier_ijk (m, 4) int, np (m,) f64)]
    into the single-GPU order and return (tier_ijk, np, budget): tier-major,
    Morton order inside a tier, and the budget accumulated as the reference
    does -- per tier numpy's pairwise sum of that tier's products, added in
    tier order (multiply.py:190-197)."""
    tij = np.concatenate([np.asarray(p[0], np.int64).reshape(-1, 4) for p in parts]) \
        if parts else np.zeros((0, 4), np.int64)
    val = np.concatenate([np.asarray(p[1], np.float64).reshape(-1) for p in parts]) \
        if parts else np.zeros(0)
    order = np.lexsort((morton_keys(tij), tij[:, 0])) if len(tij) else np.zeros(0, np.int64)
    tij, val = tij[order], val[order]
    budget = 0.0
    if len(tij):
        tiers = tij[:, 0]
        bounds = np.flatnonzero(np.r_[True, tiers[1:] != tiers[:-1], True])
        for s0, s1 in zip(bounds[:-1], bounds[1:]):
            budget += float(np.add.reduce(val[s0:s1]))
    return tij, val, budget


# -------------------------------------------------------------- collectives
class _nvtx:
    """NVTX range (torch.cuda.nvtx) around a collective or a distributed
    phase, so a profiler shows the exchanges beside the library's K1/K2/K3
    ranges; a no-op without CUDA."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        import torch

        self.on = torch.cuda.is_available()
        if self.on:
            torch.cuda.nvtx.range_push(self.name)
        return self

    def __exit__(self, *exc):
        if self.on:
            import torch

            torch.cuda.nvtx.range_pop()
        return False


class Comm:
    """The process group plus staging: NCCL works on device tensors, gloo on
    host tensors (the CPU tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def _dev(self, like):
        return like.device if self.nccl else "cpu"

    def all_gather_var(self, t):
        """All-gather tensors whose first dimension differs between ranks;
        returns the list in rank order (on t's device)."""
        with _nvtx("spamm.allgather"):
            return self._all_gather_var(t)

    def _all_gather_var(self, t):
        import torch

        dev = t.device
        x = t if self.nccl else t.cpu()
        n = torch.tensor([x.shape[0]], dtype=torch.int64, device=self._dev(t))
        ns = [torch.empty_like(n) for _ in range(self.world)]
        self.dist.all_gather(ns, n, group=self.group)
        sizes = [int(v) for v in ns]
        m = max(sizes) if sizes else 0
        if x.shape[0] < m:
            x = torch.cat([x, torch.zeros((m - x.shape[0],) + tuple(x.shape[1:]), dtype=x.dtype,
                                          device=x.device)])
        bufs = [torch.empty_like(x) for _ in range(self.world)]
        self.dist.all_gather(bufs, x.contiguous(), group=self.group)
        return [b[:s].to(dev) for b, s in zip(bufs, sizes)]

    def all_to_all_var(self, send):
        """send[q] (first dims may differ) goes to rank q; returns recv[q]
        from rank q, in rank order.  Rows of uint8 / int64 / float tensors."""
        with _nvtx("spamm.alltoall"):
            return self._all_to_all_var(send)

    def _all_to_all_var(self, send):
        import torch

        dev = send[0].device
        cnt = torch.tensor([s.shape[0] for s in send], dtype=torch.int64, device=self._dev(send[0]))
        rcnt = torch.empty_like(cnt)
        self.dist.all_to_all_single(rcnt, cnt, group=self.group)
        rsizes = [int(v) for v in rcnt]
        row = tuple(send[0].shape[1:])
        inp = torch.cat([s if self.nccl else s.cpu() for s in send]).contiguous()
        out = torch.empty((sum(rsizes),) + row, dtype=inp.dtype, device=inp.device)
        self.dist.all_to_all_single(out, inp, output_split_sizes=rsizes,
                                    input_split_sizes=[s.shape[0] for s in send],
                                    group=self.group)
        outs, o = [], 0
        for s in rsizes:
            outs.append(out[o:o + s].to(dev))
            o += s
        return outs

    def bands(self, lo, hi):
        """Every rank's [lo, hi), rank order."""
        import torch

        t = torch.tensor([[lo, hi]], dtype=torch.int64, device=self._nccl_dev())
        return [tuple(int(v) for v in b[0]) for b in self.all_gather_var(t)]

    def _nccl_dev(self):
        import torch

        return torch.device("cuda", torch.cuda.current_device()) if self.nccl else "cpu"

    def barrier(self):
        self.dist.barrier(group=self.group)


# --------------------------------------------------------- device plumbing
class DeviceArray:
    """A borrowed view of device memory exposing __cuda_array_interface__,
    so torch (NCCL collectives) can operate on a tree's storage in place."""

    def __init__(self, ptr, shape, dtype):
        self.ptr, self.shape, self.dtype = int(ptr), tuple(shape), np.dtype(dtype)

    @property
    def __cuda_array_interface__(self):
        return {"shape": self.shape, "typestr": self.dtype.str, "data": (self.ptr, False),
                "version": 3, "strides": None}


def _ptrs(tree):
    p, nsq, occ = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    _lib.check(_lib.load().spamm_tree_device_ptrs(tree._handle, ctypes.byref(p),
                                                  ctypes.byref(nsq), ctypes.byref(occ)))
    return p.value, nsq.value, occ.value


def tree_storage(tree):
    """torch view of a tree's padded N x N device storage (borrowed).  For a
    band tree only its rows (and fetched blocks) are defined."""
    import torch

    p, _, _ = _ptrs(tree)
    return torch.as_tensor(DeviceArray(p, (tree.padded_dim, tree.padded_dim), tree.dtype),
                           device=f"cuda:{tree.device}")


def _leaf_level(tree):
    """torch views of the leaf level of a tree's pyramid: (nsq f64, occ u8),
    block_grid^2 entries each, row-major."""
    import torch

    _, nsq, occ = _ptrs(tree)
    off = ((1 << (2 * tree.depth)) - 1) // 3
    G = tree.block_grid ** 2
    dev = f"cuda:{tree.device}"
    return (torch.as_tensor(DeviceArray(nsq + 8 * off, (G,), np.float64), device=dev),
            torch.as_tensor(DeviceArray(occ + off, (G,), np.uint8), device=dev))


def _to_lib(device):
    """torch's queued work (which produced data the library reads) before the
    library's stream: an event hand-off, not a device-wide synchronisation."""
    from .quadtree import torch_to_lib

    torch_to_lib(device)


def _to_torch(device):
    """The library's queued work before torch's current stream (which reads
    library output or reuses memory the library read)."""
    from .quadtree import lib_to_torch

    lib_to_torch(device)


def tree_from_padded(padded, n, leaf, device=None):
    """Adopt a padded N x N torch CUDA tensor as a tree (copied; pyramid rebuilt)."""
    import torch

    from .quadtree import _wrap

    assert padded.is_cuda and padded.is_contiguous()
    code = _lib.DTYPE_F64 if padded.dtype == torch.float64 else _lib.DTYPE_F32
    h = ctypes.c_void_p()
    dev = padded.device.index if device is None else device
    _to_lib(dev)  # torch's collectives/kernels that filled `padded` come first
    _lib.check(_lib.load().spamm_tree_from_padded_device(
        ctypes.c_void_p(padded.data_ptr()), int(n), int(padded.shape[0]), int(leaf), code, dev,
        ctypes.byref(h)))
    _to_torch(dev)  # (torch may free / reuse `padded` after the copy)
    return _wrap(h.value)


def gather_rows(local_rows, world, group=None):
    """All-gather row bands (possibly of different heights) into one array,
    rank order = row order."""
    import torch

    return torch.cat(Comm(group).all_gather_var(local_rows))


# --------------------------------------------------------- distributed trees
class ShardedTree:
    """One rank's part of a row-distributed matrix: ``tree`` is a band tree
    holding block rows ``band = (lo, hi)`` and the whole matrix's pyramid.
    Shape attributes follow QuadTreeMatrix."""

    def __init__(self, tree, band, comm):
        self.tree = tree
        self.band = (int(band[0]), int(band[1]))
        self.comm = comm
        self.logical_dim, self.leaf_size = tree.logical_dim, tree.leaf_size
        self.depth, self.padded_dim, self.dtype = tree.depth, tree.padded_dim, tree.dtype
        self.block_grid = tree.block_grid

    # -- construction -----------------------------------------------------
    @classmethod
    def from_rows(cls, rows, n, leaf, band, comm, device=None):
        """This rank's logical rows [band[0]*leaf, min(band[1]*leaf, n)) as an
        (h, >= n) torch CUDA tensor (row-major, any leading dimension)."""
        import torch

        from .quadtree import _wrap, get_device

        dev = get_device() if device is None else int(device)
        code = _lib.DTYPE_F64 if rows.dtype == torch.float64 else _lib.DTYPE_F32
        if rows.numel():
            assert rows.is_cuda and rows.stride(1) == 1
        _to_lib(dev)
        h = ctypes.c_void_p()
        ld = int(rows.stride(0)) if rows.numel() else int(n)
        _lib.check(_lib.load().spamm_tree_band_from_device(
            ctypes.c_void_p(rows.data_ptr() if rows.numel() else 0), int(n), max(ld, int(n)),
            int(leaf), code, int(band[0]), int(band[1]), dev, ctypes.byref(h)))
        _to_torch(dev)
        st = cls(_wrap(h.value), band, comm)
        st.gather_pyramid()
        return st

    @classmethod
    def scatter(cls, full, n, leaf, comm, src=0, weights=None, dtype=None):
        """Distribute a matrix held by rank `src` (an (n, n) or padded torch
        CUDA tensor there; ignored elsewhere) by block rows: each rank receives
        only its band's rows (NCCL point-to-point from `src`) -- n^2 s / W
        bytes per rank -- then builds its band tree and the shared pyramid."""
        import torch

        nb = padded_blocks(n, leaf)
        bands = [row_shard(r, comm.world, n, leaf, weights) for r in range(comm.world)]
        lo, hi = bands[comm.rank]
        tdt = dtype or (full.dtype if full is not None else torch.float64)
        dev = comm._nccl_dev()
        mine = None
        if comm.rank == src:
            for r, (a, b) in enumerate(bands):
                r0, r1 = min(a * leaf, n), min(b * leaf, n)
                part = full[r0:r1, :n].contiguous()
                if r == src:
                    mine = part
                elif r1 > r0:
                    comm.dist.send(part if comm.nccl else part.cpu(), dst=r, group=comm.group)
        else:
            r0, r1 = min(lo * leaf, n), min(hi * leaf, n)
            buf = torch.empty((r1 - r0, n), dtype=tdt, device=dev)
            if r1 > r0:
                comm.dist.recv(buf, src=src, group=comm.group)
            mine = buf
        if not mine.is_cuda:
            mine = mine.cuda()
        del nb
        return cls.from_rows(mine, n, leaf, (lo, hi), comm)

    @classmethod
    def from_product(cls, tree, band, comm):
        """Adopt a row-shard product (band tree with the band's own pyramid)."""
        _lib.check(_lib.load().spamm_tree_band_set(tree._handle, int(band[0]), int(band[1])))
        st = cls(tree, band, comm)
        st.gather_pyramid()
        return st

    # -- pyramids ---------------------------------------------------------
    def gather_pyramid(self, tree=None):
        """All-gather the leaf level of `tree` (default: this band tree) across
        the ranks' bands and rebuild the pyramid above it on every rank."""
        tree = self.tree if tree is None else tree
        gather_leaf_level(tree, self.band, self.comm)

    # -- queries ----------------------------------------------------------
    def norm(self):
        return self.tree.norm()

    def _root_norm_sq(self):
        return self.tree._root_norm_sq

    def trace(self):
        """Tr over the logical diagonal, summed exactly as the single-GPU
        trace (numpy add.reduce over the whole diagonal, quadtree.py:274-277):
        each rank reads its rows' diagonal, the pieces are all-gathered."""
        import torch

        lo, hi = self.band
        n, leaf = self.logical_dim, self.leaf_size
        r0, r1 = min(lo * leaf, n), min(hi * leaf, n)
        d = np.empty(max(r1 - r0, 0), dtype=self.dtype)
        if r1 > r0:
            _lib.check(_lib.load().spamm_tree_diagonal_rows(self.tree._handle, lo, hi,
                                                            d.ctypes.data))
        t = torch.from_numpy(d.view(np.uint8).copy()).to(self.comm._nccl_dev())
        full = torch.cat(self.comm.all_gather_var(t)).cpu().numpy().view(self.dtype)
        return float(np.add.reduce(full))

    def rows_tensor(self):
        """torch view of this band's padded rows (h x N), on the device."""
        lo, hi = self.band
        return tree_storage(self.tree)[lo * self.leaf_size:hi * self.leaf_size]

    def gather_padded(self):
        """The whole padded matrix on every rank (torch CUDA tensor): each
        band's rows, with its empty blocks zero-filled, all-gathered.  For
        checks and small matrices; the multiply never needs it."""
        import torch

        lo, hi = self.band
        L, N = self.leaf_size, self.padded_dim
        rows = self.rows_tensor().clone()
        occ = _leaf_level(self.tree)[1].view(self.block_grid, self.block_grid)[lo:hi]
        mask = occ.bool().repeat_interleave(L, 0).repeat_interleave(L, 1)
        rows[~mask] = 0
        return torch.cat(self.comm.all_gather_var(rows)).view(N, N)

    def gather_dense(self):
        """The logical n x n matrix on every rank, as numpy (to_dense())."""
        n = self.logical_dim
        return self.gather_padded()[:n, :n].cpu().numpy()


def gather_leaf_level(tree, band, comm):
    """Leaf-level (norm, occupancy) all-gather of a band tree, then the
    pyramid above it (spamm_tree_pyramid_rebuild): bit-identical on every
    rank to the pyramid of the whole matrix."""
    import torch

    nsq, occ = _leaf_level(tree)
    _to_torch(tree.device)  # the library's leaf level before torch reads it
    nb = tree.block_grid
    lo, hi = band
    mine = torch.cat([nsq[lo * nb:hi * nb].view(torch.uint8).view(-1, 8),
                      occ[lo * nb:hi * nb].view(-1, 1)], dim=1)  # 9 bytes per leaf
    parts = comm.all_gather_var(mine)
    full = torch.cat(parts).to(nsq.device)
    assert full.shape[0] == nb * nb, "bands must cover every block row"
    nsq.copy_(full[:, :8].contiguous().view(torch.float64).view(-1))
    occ.copy_(full[:, 8])
    _to_lib(tree.device)  # torch's writes of the leaf level before the rebuild
    _lib.check(_lib.load().spamm_tree_pyramid_rebuild(tree._handle))
    tree._host_pyramid = None
    info = _lib.TreeInfo()
    _lib.check(_lib.load().spamm_tree_info_get(tree._handle, ctypes.byref(info)))
    tree._root_nsq = float(info.root_norm_sq)
    tree._root = None


def halo_exchange(b, needed, comm):
    """Fetch into b's storage the listed blocks (ids k * nb + j, any order)
    that other ranks hold: ids to their owners (all-to-all), blocks back
    (all-to-all).  Returns the bytes this rank received."""
    with _nvtx("spamm.halo_exchange"):
        return _halo_exchange(b, needed, comm)


def _halo_exchange(b, needed, comm):
    import torch

    nb, L = b.block_grid, b.leaf_size
    esz = np.dtype(b.dtype).itemsize
    blk = L * L * esz
    bands = comm.bands(*b.band)
    owner_of_row = np.zeros(nb, np.int64)
    for r, (lo, hi) in enumerate(bands):
        owner_of_row[lo:hi] = r
    needed = np.unique(np.asarray(needed, np.int64))
    needed = needed[owner_of_row[needed // nb] != comm.rank] if len(needed) else needed
    owners = owner_of_row[needed // nb] if len(needed) else needed
    dev = comm._nccl_dev()
    req = [torch.from_numpy(needed[owners == q]).to(dev) for q in range(comm.world)]
    asked = comm.all_to_all_var(req)               # ids other ranks want from me
    L_ = _lib.load()
    send = []
    for q in range(comm.world):
        ids = asked[q].to(f"cuda:{b.tree.device}")
        buf = torch.empty((ids.numel(), blk), dtype=torch.uint8, device=f"cuda:{b.tree.device}")
        if ids.numel():
            _to_lib(b.tree.device)
            _lib.check(L_.spamm_tree_blocks_gather_device(b.tree._handle,
                                                          ctypes.c_void_p(ids.data_ptr()),
                                                          ids.numel(),
                                                          ctypes.c_void_p(buf.data_ptr())))
            _to_torch(b.tree.device)
        send.append(buf if comm.nccl else buf.cpu())
    got = comm.all_to_all_var(send)                # the blocks I asked for
    ids = torch.cat([r.to(f"cuda:{b.tree.device}") for r in req])
    data = torch.cat([g.to(f"cuda:{b.tree.device}") for g in got])
    if ids.numel():
        _to_lib(b.tree.device)
        _lib.check(L_.spamm_tree_blocks_scatter_device(b.tree._handle,
                                                       ctypes.c_void_p(ids.data_ptr()),
                                                       ids.numel(),
                                                       ctypes.c_void_p(data.data_ptr())))
    b.tree._host_padded = None
    return int(data.numel())


def reduce_stats(stats, group=None):
    """Sum per-rank ProductStats (or dicts) over the group: integers exactly,
    max_depth_reached as the max, budgets added in rank order.  (The budget
    then equals the single-GPU one to rounding; spamm_sharded rebuilds it bit
    for bit from the pruned calls instead.)"""
    import torch

    comm = Comm(group)
    keys = ("leaf_matmuls", "pruned_calls", "pruned_volume", "empty_skip_volume")
    get = (lambda k: stats[k]) if isinstance(stats, dict) else (lambda k: getattr(stats, k))
    ints = torch.tensor([[get(k) for k in keys] + [get("max_depth_reached")]], dtype=torch.int64,
                        device=comm._nccl_dev())
    flo = torch.tensor([[get("omitted_budget")]], dtype=torch.float64, device=comm._nccl_dev())
    all_i = torch.cat(comm.all_gather_var(ints)).cpu()
    all_f = torch.cat(comm.all_gather_var(flo)).cpu()
    out = {k: int(all_i[:, q].sum()) for q, k in enumerate(keys)}
    out["max_depth_reached"] = int(all_i[:, len(keys)].max())
    budget = 0.0
    for v in all_f[:, 0].tolist():  # fixed rank order
        budget += v
    out["omitted_budget"] = budget
    return out


def spamm_sharded(a, b, config=None, keep_triples=False):
    """C = spamm(A, B) with A, B row-distributed ShardedTrees: this rank
    computes C's block rows in its band.  Returns (C ShardedTree,
    ProductStats, detail) -- every ProductStats field (boxes in reference
    order and the budget included) equal to the single-GPU multiply's, C's
    pyramid the single-GPU C's bit for bit, and C's band rows the single-GPU
    rows bit for bit.  detail: this rank's MultiplyDetail plus ``halo_bytes``."""
    import torch

    from .multiply import ProductStats, PrunedBox, SpammConfig, spamm_detailed
    from .quadtree import _require_conformable

    if config is None:
        config = SpammConfig()
    _require_conformable(a, b)
    comm = a.comm
    lo, hi = a.band
    assert b.band == a.band, "operands must share the row partition"
    nb = a.block_grid
    halo = 0
    if comm.world == 1:
        # one rank holds every row: no exchange, its statistics are the global ones
        c_tree, st, det = spamm_detailed(a.tree, b.tree, config, keep_triples=keep_triples,
                                         rows=(lo, hi))
        c = ShardedTree.from_product(c_tree, (lo, hi), comm)
        if det is not None:
            det.halo_bytes = 0
        return c, st, det
    if hi > lo:
        # plan: the B blocks this band's retained triples read
        # (a bitmask over the block grid formed on the device: no triples copied)
        _, _, plan = spamm_detailed(a.tree, b.tree, replace_cfg(config), rows=(lo, hi),
                                    traverse_only=True, need_blocks=True)
        needed = np.flatnonzero(plan.need_blocks).astype(np.int64)
    else:
        needed = np.zeros(0, np.int64)
    halo = halo_exchange(b, needed, comm)
    if hi > lo:
        c_tree, st, det = spamm_detailed(a.tree, b.tree, config, keep_triples=keep_triples,
                                         rows=(lo, hi), keep_pruned=config.count_stats)
    else:  # an empty band still joins every collective
        c_tree = _empty_band(a)
        st, det = ProductStats(boxes=[] if config.collect_boxes else None), None
    c = ShardedTree.from_product(c_tree, (lo, hi), comm)
    # statistics: integers summed, the pruned calls merged into reference order
    keys = ("leaf_matmuls", "pruned_calls", "pruned_volume", "empty_skip_volume")
    dev = comm._nccl_dev()
    ints = torch.tensor([[getattr(st, k) for k in keys] + [st.max_depth_reached]],
                        dtype=torch.int64, device=dev)
    all_i = torch.cat(comm.all_gather_var(ints)).cpu()
    out = ProductStats(boxes=[] if config.collect_boxes else None)
    for q, k in enumerate(keys):
        setattr(out, k, int(all_i[:, q].sum()))
    out.max_depth_reached = int(all_i[:, len(keys)].max())
    if config.count_stats or config.collect_boxes:
        pr = det.pruned if det is not None and det.pruned is not None else np.zeros((0, 4), np.int32)
        pv = det.pruned_np if det is not None and det.pruned_np is not None else np.zeros(0)
        t_ijk = comm.all_gather_var(torch.from_numpy(np.ascontiguousarray(pr, np.int64)).to(dev))
        t_np = comm.all_gather_var(torch.from_numpy(np.ascontiguousarray(pv, np.float64)).to(dev))
        tij, _, budget = merge_pruned([(x.cpu().numpy(), y.cpu().numpy())
                                       for x, y in zip(t_ijk, t_np)])
        if config.count_stats:
            out.omitted_budget = budget
        if config.collect_boxes:
            N = a.padded_dim
            out.boxes = [PrunedBox(int(i) * (N >> int(t)), int(j) * (N >> int(t)),
                                   int(k) * (N >> int(t)), N >> int(t), int(t))
                         for t, i, j, k in tij.tolist()]
    if det is not None:
        det.halo_bytes = halo
    return c, out, det


def replace_cfg(config):
    """The plan pass needs no statistics, boxes or pruned records."""
    from dataclasses import replace

    return replace(config, collect_boxes=False, count_stats=False)


def _empty_band(like):
    """A band tree with no rows (a rank with an empty range)."""
    from .quadtree import _wrap

    code = _lib.DTYPE_F64 if like.dtype == np.float64 else _lib.DTYPE_F32
    h = ctypes.c_void_p()
    _lib.check(_lib.load().spamm_tree_band_from_device(
        None, like.logical_dim, like.logical_dim, like.leaf_size, code, like.band[0],
        like.band[0], like.tree.device, ctypes.byref(h)))
    return _wrap(h.value)


# ------------------------------------------------------------ sharded TC2
def tc2_initial_guess_sharded(f):
    """X0 = (eps_max I - F) / (eps_max - eps_min) with Gershgorin bounds
    (purification.py:77-92) on a row-distributed F: each rank bounds its
    rows, min / max are combined exactly, and X0's band rows are formed with
    the reference's element-wise expression."""
    import torch

    from .purification import HOST_DENSE_MAX

    lo, hi = f.band
    n, L = f.logical_dim, f.leaf_size
    r0, r1 = min(lo * L, n), min(hi * L, n)
    if n <= HOST_DENSE_MAX:
        return _initial_guess_host(f, r0, r1)
    rows = f.rows_tensor()[:r1 - r0, :n].to(torch.float64)
    occ = _leaf_level(f.tree)[1].view(f.block_grid, f.block_grid)[lo:hi]
    mask = occ.bool().repeat_interleave(L, 0).repeat_interleave(L, 1)[:r1 - r0, :n]
    rows = torch.where(mask, rows, torch.zeros_like(rows))  # (empty blocks are not held)
    idx = torch.arange(r0, r1, device=rows.device)
    c = rows[torch.arange(r1 - r0, device=rows.device), idx] if r1 > r0 else rows.new_zeros(0)
    r = rows.abs().sum(dim=1) - c.abs()
    inf = torch.tensor(float("inf"), dtype=torch.float64, device=rows.device)
    lo_b = (c - r).min() if r1 > r0 else inf
    hi_b = (c + r).max() if r1 > r0 else -inf
    dev = f.comm._nccl_dev()
    b = torch.cat(f.comm.all_gather_var(torch.stack([lo_b, -hi_b]).view(1, 2).to(dev))).cpu()
    emin, emax = float(b[:, 0].min()), -float(b[:, 1].min())
    if emax == emin:
        x = torch.zeros_like(rows)
        x[torch.arange(r1 - r0, device=rows.device), idx] = 0.5
    else:
        eye = torch.zeros_like(rows)
        eye[torch.arange(r1 - r0, device=rows.device), idx] = 1.0
        x = (emax * eye - rows) / (emax - emin)
    x = x.to(torch.float32 if f.dtype == np.float32 else torch.float64).contiguous()
    return ShardedTree.from_rows(x, n, L, f.band, f.comm)


def _initial_guess_host(f, r0, r1):
    """The band's rows of X0 with the single-GPU driver's numpy expressions
    (row sums per row, then (hi I - F) / (hi - lo) element-wise): each row's
    values depend only on that row and the global bounds, so the band's rows
    are the whole matrix's rows bit for bit."""
    import torch

    n, L = f.logical_dim, f.leaf_size
    lo, hi = f.band
    rows = f.rows_tensor()[:r1 - r0, :n]
    occ = _leaf_level(f.tree)[1].view(f.block_grid, f.block_grid)[lo:hi]
    mask = occ.bool().repeat_interleave(L, 0).repeat_interleave(L, 1)[:r1 - r0, :n]
    fd = torch.where(mask, rows, torch.zeros_like(rows)).cpu().numpy().astype(np.float64)
    q = np.arange(r1 - r0)
    c = fd[q, r0 + q]
    r = np.abs(fd).sum(axis=1) - np.abs(c)
    mine = np.array([[(c - r).min() if len(c) else np.inf, -((c + r).max() if len(c) else -np.inf)]])
    dev = f.comm._nccl_dev()
    b = torch.cat(f.comm.all_gather_var(torch.from_numpy(mine).to(dev))).cpu().numpy()
    emin, emax = float(b[:, 0].min()), -float(b[:, 1].min())
    eye = np.zeros_like(fd)
    eye[q, r0 + q] = 1.0
    x0 = 0.5 * eye if emax == emin else (emax * eye - fd) / (emax - emin)
    x0 = torch.from_numpy(np.ascontiguousarray(x0.astype(f.dtype))).cuda(f.tree.device)
    return ShardedTree.from_rows(x0, n, L, f.band, f.comm)


def _tc2_pass(x, x2, make_y):
    """The fused band pass plus the gathers that make its outputs global:
    returns (y ShardedTree or None, d_root_nsq, e_root_nsq)."""
    from .quadtree import tc2_update

    y, d, e, _, _ = tc2_update(x.tree, x2.tree, make_y, rows=x.band)
    gather_leaf_level(d, x.band, x.comm)
    d_root = d._root_nsq
    e_root = 0.0
    ys = None
    if make_y:
        gather_leaf_level(e, x.band, x.comm)
        e_root = e._root_nsq
        ys = ShardedTree(y, x.band, x.comm)
        ys.gather_pyramid()
    return ys, d_root, e_root


def tc2_step_sharded(x, n_occ, mode):
    """One TC2 sweep on a row-distributed iterate (purification.py:105-134);
    returns (next, ProductStats, displacement ||next - X||_F) -- the values
    of the single-GPU sweep, bit for bit."""
    from .multiply import SpammConfig
    from .purification import _FIXED_POINT_FACTOR, DroppingMode, SpammMode

    tr = x.trace()
    if isinstance(mode, SpammMode):
        x2, stats, _ = spamm_sharded(x, x, SpammConfig(tau=mode.tau))
    elif isinstance(mode, DroppingMode) and mode.tau == 0:
        x2, stats, _ = spamm_sharded(x, x, SpammConfig(tau=0.0))
    else:
        raise TypeError(f"sharded purification supports SpammMode (and DroppingMode(0)), got {mode!r}")
    y, d_nsq, e_nsq = _tc2_pass(x, x2, make_y=not tr >= n_occ)  # NaN trace: 2X - X^2
    gap = float(np.sqrt(d_nsq))
    if gap <= _FIXED_POINT_FACTOR * np.finfo(x.dtype).eps * x.logical_dim:
        return x, stats, 0.0
    if tr >= n_occ:
        return x2, stats, gap
    return y, stats, float(np.sqrt(e_nsq))


def purify_sharded(f, n_occ, mode, max_iter=50, reference_energy=None):
    """purify() (purification.py:150-227) on a row-distributed Hamiltonian:
    the same latch and accounting, every sweep through tc2_step_sharded; the
    density stays distributed.  Energies are Tr(P F) from the gathered dense
    matrices up to purification.HOST_DENSE_MAX (the single-GPU driver's
    numpy expression, bit for bit), above it from per-band device partial
    sums added in rank order."""
    import torch

    from .purification import (_TERMINAL_GAP, HOST_DENSE_MAX, PurificationResult, SpammMode)

    if max_iter < 1:
        raise ValueError(f"max_iter must be >= 1, got {max_iter}")
    if mode.tau < 0 or not math.isfinite(mode.tau):
        raise ValueError(f"mode.tau must be finite and >= 0, got {mode.tau}")
    n = f.logical_dim
    if not 0 <= n_occ <= n:
        raise ValueError(f"n_occ must be in [0, {n}], got {n_occ}")
    if n <= HOST_DENSE_MAX:
        fd = f.gather_dense()
        if not np.array_equal(fd, fd.T):
            raise ValueError("purification requires a symmetric matrix")
    x = tc2_initial_guess_sharded(f)
    traces = [x.trace()]
    counts = []
    best_x, best_gap = None, math.inf
    held, held_stats = False, None
    with np.errstate(over="ignore", invalid="ignore"):
        for _ in range(max_iter):
            if held_stats is not None:
                counts.append(held_stats.leaf_matmuls)
                traces.append(traces[-1])
                continue
            nxt, stats, gap = tc2_step_sharded(x, n_occ, mode)
            counts.append(stats.leaf_matmuls)
            if held:
                held_stats = stats
                traces.append(traces[-1])
                continue
            if gap < best_gap:
                best_gap, best_x, x = gap, x, nxt
            elif best_gap <= _TERMINAL_GAP and gap > 4.0 * best_gap:
                x, held = best_x, True
            else:
                x = nxt
            traces.append(x.trace())
    if n <= HOST_DENSE_MAX:
        energy = float(np.einsum("ij,ji->", x.gather_dense().astype(np.float64),
                                 f.gather_dense().astype(np.float64)))
    else:  # Tr(P F) = sum over this band's rows of P_ij F_ji = sum P_ij F_ij (F symmetric)
        lo, hi = x.band
        L = x.leaf_size
        r0, r1 = min(lo * L, n), min(hi * L, n)
        p = x.rows_tensor()[:r1 - r0, :n].to(torch.float64)
        fr = f.rows_tensor()[:r1 - r0, :n].to(torch.float64)
        mp = _leaf_level(x.tree)[1].view(x.block_grid, -1)[lo:hi].bool()
        mf = _leaf_level(f.tree)[1].view(f.block_grid, -1)[lo:hi].bool()
        m = (mp & mf).repeat_interleave(L, 0).repeat_interleave(L, 1)[:r1 - r0, :n]
        part = torch.where(m, p * fr, torch.zeros_like(p)).sum().view(1, 1)
        energy = 0.0
        for v in torch.cat(x.comm.all_gather_var(part.to(x.comm._nccl_dev()))).cpu()[:, 0].tolist():
            energy += v
    if mode.tau == 0:
        ref, delta = energy, 0.0
    else:
        ref = (float(reference_energy) if reference_energy is not None
               else purify_sharded(f, n_occ, SpammMode(0.0), max_iter=max_iter).energy)
        diff = abs(energy - ref)
        delta = (0.0 if diff == 0 else math.inf) if ref == 0 else diff / abs(ref)
    total = int(sum(counts))
    return PurificationResult(density=x, iterations=max_iter, total_leaf_matmuls=total,
                              avg_leaf_matmuls=total / max_iter, energy=energy,
                              delta_e_rel=delta, reference_energy=ref,
                              trace_history=traces, step_leaf_matmuls=counts)
