"""Device-resident quadtree matrices (drop-in for ``spamm.quadtree``).

A tree owns, on one B200, the zero-padded ``leaf_size * 2**depth`` square
(row-major), a squared-Frobenius-norm pyramid and an occupancy pyramid, all
built by the CUDA library (K1, ``csrc/tree.cu``).  The reference keeps the
same three things as numpy arrays (quadtree.py:116-151); here they are
mirrored to the host lazily, only when a caller reads the private
attributes (``_padded``, ``_blocks``, ``_leaf_nonzero``, ``_norm_sq``,
``_occupied``) or walks ``root`` -- so code written against the reference's
white-box attributes keeps working.

Reference: arxiv/paper_1011_3534, pkg/src/spamm/quadtree.py.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib

_SUPPORTED_DTYPES = (np.dtype(np.float64), np.dtype(np.float32))  # quadtree.py:18
_QUADRANTS = ((0, 0), (0, 1), (1, 0), (1, 1))                       # quadtree.py:22

_default_device = None


def set_device(device):
    """Select the CUDA ordinal new trees are built on (default: $SPAMM_DEVICE,
    else $LOCAL_RANK, else 0)."""
    global _default_device
    _default_device = int(device)


def get_device():
    if _default_device is not None:
        return _default_device
    return int(os.environ.get("SPAMM_DEVICE", os.environ.get("LOCAL_RANK", "0")))


class DimensionMismatchError(ValueError):
    """Non-square input, or two trees that are not conformable
    (quadtree.py:26-28)."""


class EmptyNode:
    """An exactly-zero submatrix (quadtree.py:31-39); one shared instance."""

    __slots__ = ()
    kind = "empty"
    norm_sq = 0.0

    def __repr__(self):
        return "EmptyNode()"


EMPTY = EmptyNode()


class LeafNode:
    """A dense leaf block, a read-only view into the host mirror (quadtree.py:45-56)."""

    __slots__ = ("block", "norm_sq")
    kind = "leaf"

    def __init__(self, block, norm_sq):
        self.block = block
        self.norm_sq = norm_sq

    def __repr__(self):
        return f"LeafNode(norm_sq={self.norm_sq!r})"


class InteriorNode:
    """Four children in quadrant order 11, 12, 21, 22 (quadtree.py:59-71)."""

    __slots__ = ("children", "norm_sq")
    kind = "interior"

    def __init__(self, children, norm_sq):
        self.children = children
        self.norm_sq = norm_sq

    def __repr__(self):
        return "InteriorNode([%s], norm_sq=%r)" % (",".join(c.kind for c in self.children),
                                                   self.norm_sq)


class PendingBlocks:
    """An in-flight ``nonzero_blocks(wait=False)`` copy.  ``wait()`` blocks
    until the blocks are in host memory and returns ``(ids, blocks)``; an
    unwaited transfer is waited for when the object is collected (the host
    buffer must outlive the copy)."""

    def __init__(self, handle, ids, blocks):
        self._handle = handle
        self.ids = ids
        self.blocks = blocks

    def wait(self):
        h, self._handle = self._handle, None
        if h is not None:
            _lib.check(_lib.load().spamm_transfer_wait(h))
        return self.ids, self.blocks

    def __del__(self):
        if getattr(self, "_handle", None) is not None:
            try:
                self.wait()
            except Exception:  # interpreter shutdown
                pass


def _level_slices(depth):
    out, off = [], 0
    for k in range(depth + 1):
        out.append((off, 1 << k))
        off += 1 << (2 * k)
    return out


class QuadTreeMatrix:
    """Immutable quadtree matrix living on a CUDA device.

    Public attributes match the reference (quadtree.py:95-113):
    ``logical_dim``, ``leaf_size``, ``depth``, ``padded_dim``, ``dtype``,
    plus ``block_grid``, ``element_precision``, ``root``, ``norm()``,
    ``to_dense()`` and ``structurally_equal()``.  ``device`` names the GPU.
    """

    def __init__(self, handle=None, _internal=False):
        if not _internal:
            raise TypeError("use from_dense() to construct a QuadTreeMatrix")
        self._handle = ctypes.c_void_p(handle)
        info = _lib.TreeInfo()
        _lib.check(_lib.load().spamm_tree_info_get(self._handle, ctypes.byref(info)))
        self.logical_dim = int(info.logical_dim)
        self.leaf_size = int(info.leaf_size)
        self.depth = int(info.depth)
        self.padded_dim = int(info.padded_dim)
        self.dtype = _SUPPORTED_DTYPES[info.dtype]
        self.device = int(info.device)
        self._root_nsq = float(info.root_norm_sq)
        self._pending = False  # an asynchronous build (from_dense(wait=False))
        self._src = None       # ... and the host array it reads
        self._host_padded = None
        self._host_pyramid = None
        self._root = None

    @property
    def _root_norm_sq(self):
        if self._pending:
            self.wait()
        return self._root_nsq

    def wait(self):
        """Block until an asynchronous build (``from_dense(wait=False)``) is
        complete; returns the tree.  A no-op for every other tree."""
        if self._pending:
            L = _lib.load()
            _lib.check(L.spamm_tree_wait(self._handle))
            info = _lib.TreeInfo()
            _lib.check(L.spamm_tree_info_get(self._handle, ctypes.byref(info)))
            self._root_nsq = float(info.root_norm_sq)
            self._pending = False
            self._src = None
        return self

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            try:
                # (a pending build is waited for inside: it may read _src)
                _lib.load().spamm_tree_free(h)
            except Exception:  # interpreter shutdown
                pass
            self._handle = None

    # -- structure ----------------------------------------------------------
    @property
    def block_grid(self):
        return self.padded_dim // self.leaf_size

    @property
    def element_precision(self):
        return "double" if self.dtype == np.float64 else "single"

    @property
    def root(self):
        """Root node of the node view (quadtree.py:164-180), built lazily."""
        if self._root is None:
            self._root = self._node(0, 0, 0)
        return self._root

    def _node(self, tier, qi, qj):
        if not self._occupied[tier][qi, qj]:
            return EMPTY
        nsq = float(self._norm_sq[tier][qi, qj])
        if tier == self.depth:
            return LeafNode(self._blocks[qi, qj], nsq)
        kids = tuple(self._node(tier + 1, 2 * qi + di, 2 * qj + dj) for di, dj in _QUADRANTS)
        return InteriorNode(kids, nsq)

    # -- lazily mirrored host state (white-box attributes) --------------------
    @property
    def _padded(self):
        if self._host_padded is None:
            out = np.empty((self.padded_dim, self.padded_dim), dtype=self.dtype)
            _lib.check(_lib.load().spamm_tree_padded_to_host(self._handle, out.ctypes.data))
            out.flags.writeable = False
            self._host_padded = out
        return self._host_padded

    @property
    def _blocks(self):
        nb, b = self.block_grid, self.leaf_size
        return self._padded.reshape(nb, b, nb, b).swapaxes(1, 2)

    def _pyramid(self):
        if self._host_pyramid is None:
            size = ((1 << (2 * (self.depth + 1))) - 1) // 3
            nsq = np.empty(size, np.float64)
            occ = np.empty(size, np.uint8)
            _lib.check(_lib.load().spamm_tree_pyramid_to_host(self._handle, nsq.ctypes.data,
                                                               occ.ctypes.data))
            levels_n, levels_o = [], []
            for off, side in _level_slices(self.depth):
                a = nsq[off:off + side * side].reshape(side, side)
                o = occ[off:off + side * side].reshape(side, side).astype(bool)
                a.flags.writeable = False
                o.flags.writeable = False
                levels_n.append(a)
                levels_o.append(o)
            self._host_pyramid = (levels_n, levels_o, nsq, occ)
        return self._host_pyramid

    @property
    def _norm_sq(self):
        return self._pyramid()[0]

    @property
    def _occupied(self):
        return self._pyramid()[1]

    @property
    def _leaf_nonzero(self):
        return self._occupied[self.depth]

    # -- queries --------------------------------------------------------------
    def nonzero_blocks(self, out=None, wait=True):
        """(ids, blocks): the tree's nonzero leaves -- the reference's
        ``_blocks[_leaf_nonzero]`` with their indices i * block_grid + j in
        ascending order -- read back in one transfer (extension: the product
        without its empty blocks).  ``out``: optional C-contiguous
        (>= count, b, b) host array of the tree's dtype (e.g. pinned).

        ``wait=False`` returns a :class:`PendingBlocks` at once: the copy runs
        on a separate copy-out stream and overlaps the caller's next calls
        (pass pinned ``out`` for that); ``.wait()`` yields ``(ids, blocks)``."""
        occ = np.asarray(self._occupied[self.depth]).reshape(-1)
        ids = np.flatnonzero(occ).astype(np.int64)
        b = self.leaf_size
        if out is None:
            out = np.empty((len(ids), b, b), dtype=self.dtype)
        elif (out.dtype != self.dtype or out.ndim != 3 or out.shape[1:] != (b, b)
              or out.shape[0] < len(ids) or not out.flags.c_contiguous):
            raise ValueError("out must be a C-contiguous (>= count, b, b) array of the tree dtype")
        # ids=NULL below: the device lists the nonzero leaves itself (the same
        # ones as `ids`, both from the occupancy pyramid)
        if not wait:
            h = ctypes.c_void_p()
            _lib.check(_lib.load().spamm_tree_blocks_to_host_async(
                self._handle, None, len(ids), out.ctypes.data, ctypes.byref(h)))
            return PendingBlocks(h, ids, out[:len(ids)])
        _lib.check(_lib.load().spamm_tree_blocks_to_host(self._handle, None, len(ids),
                                                         out.ctypes.data))
        return ids, out[:len(ids)]

    def to_dense(self, out=None):
        """Fresh n x n host array with the padding stripped (quadtree.py:184-187).

        ``out`` (extension): an existing C-contiguous n x n host array of the
        tree's dtype to copy into -- e.g. pinned memory for fast transfers.
        """
        n = self.logical_dim
        if out is None:
            out = np.empty((n, n), dtype=self.dtype)
        elif (out.shape != (n, n) or out.dtype != self.dtype
              or not out.flags.c_contiguous or not out.flags.writeable):
            raise ValueError("out must be a writeable C-contiguous (n, n) array of the tree dtype")
        _lib.check(_lib.load().spamm_tree_to_host(self._handle, out.ctypes.data, n))
        return out

    def norm(self):
        """sqrt of the root's cached squared norm (quadtree.py:189-191)."""
        return float(np.sqrt(self._root_norm_sq))

    def structurally_equal(self, other):
        """Same shape, occupancy and bit-identical storage (quadtree.py:193-202)."""
        if not isinstance(other, QuadTreeMatrix):
            return False
        return (self.logical_dim == other.logical_dim
                and self.leaf_size == other.leaf_size
                and self.dtype == other.dtype
                and np.array_equal(self._leaf_nonzero, other._leaf_nonzero)
                and self._padded.tobytes() == other._padded.tobytes())

    def __repr__(self):
        return (f"QuadTreeMatrix(n={self.logical_dim}, leaf={self.leaf_size}, "
                f"depth={self.depth}, norm={self.norm():.6g})")


def _require_conformable(a, b):
    """quadtree.py:209-215."""
    if a.logical_dim != b.logical_dim or a.leaf_size != b.leaf_size:
        raise DimensionMismatchError(
            f"trees not conformable: ({a.logical_dim}, leaf {a.leaf_size}) vs "
            f"({b.logical_dim}, leaf {b.leaf_size})")
    if a.dtype != b.dtype:
        raise DimensionMismatchError(f"dtype mismatch: {a.dtype} vs {b.dtype}")


def _wrap(handle):
    return QuadTreeMatrix(handle, _internal=True)


def from_dense(dense, leaf_size=4, dtype=None, device=None, wait=True):
    """Build a device quadtree from a dense square array (quadtree.py:218-251).

    Validation and exception types follow the reference; the padding, the
    leaf norms and the pyramid are computed on the GPU.

    ``wait=False`` (extension): return at once; the host->device copy and
    the pyramid run on a separate copy-in stream, overlapping work already
    queued (e.g. the previous matrix's multiplies).  Every later call on the
    tree is ordered after the build.  Pass pinned host memory for the copy to
    be truly asynchronous; the tree keeps a reference to the array until
    ``wait()`` (or its first host-side use of the root norm).
    """
    if leaf_size < 1 or (leaf_size & (leaf_size - 1)) != 0:
        raise ValueError(f"leaf_size must be a power of two >= 1, got {leaf_size}")
    target = np.dtype(np.float64) if dtype is None else np.dtype(dtype)
    if target not in _SUPPORTED_DTYPES:
        raise ValueError(f"unsupported element dtype {target}")
    arr = np.asarray(dense, dtype=target)
    if arr.ndim != 2 or arr.shape[0] != arr.shape[1]:
        raise DimensionMismatchError(f"expected a square 2-D array, got shape {arr.shape}")
    n = arr.shape[0]
    if n < 1:
        raise ValueError("matrix dimension must be >= 1")
    arr = np.ascontiguousarray(arr)
    h = ctypes.c_void_p()
    dev = get_device() if device is None else int(device)
    code = _lib.DTYPE_F64 if target == np.float64 else _lib.DTYPE_F32
    if not wait:
        _lib.check(_lib.load().spamm_tree_from_host_async(arr.ctypes.data, n, n, int(leaf_size),
                                                          code, dev, ctypes.byref(h)))
        t = _wrap(h.value)
        t._pending = True
        t._src = arr
        return t
    _lib.check(_lib.load().spamm_tree_from_host(arr.ctypes.data, n, n, int(leaf_size), code,
                                                dev, ctypes.byref(h)))
    return _wrap(h.value)


def torch_stream(device):
    """The handle of torch's current CUDA stream on `device` (0 = the legacy
    stream, also when torch is not in use): the stream a caller's device data
    is produced / consumed on."""
    import sys

    torch = sys.modules.get("torch")
    if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
        return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    return ctypes.c_void_p(0)


def torch_to_lib(device):
    """Stream hand-off: the library's stream waits for the work torch has
    queued so far (torch produced data the library reads).  An event wait on
    the device, not a device-wide synchronisation."""
    _lib.check(_lib.load().spamm_stream_wait(int(device), torch_stream(device)))


def lib_to_torch(device):
    """Stream hand-off: torch's current stream waits for the library's queued
    work (torch reads library results or reuses memory the library read)."""
    _lib.check(_lib.load().spamm_stream_signal(int(device), torch_stream(device)))


def from_device_pointer(ptr, n, leaf_size=4, dtype=np.float64, device=None, ld=None, stream=None):
    """Build a tree from an n x n array already resident in device memory
    (e.g. a torch CUDA tensor's ``data_ptr()``); no host staging.  Stream
    ordered (spamm_tree_from_device_on): the copy starts after the work
    queued on `stream` (default: torch's current stream) and that stream
    waits for the copy, so the caller may free or reuse the array in stream
    order -- no device-wide synchronisation."""
    target = np.dtype(dtype)
    if target not in _SUPPORTED_DTYPES:
        raise ValueError(f"unsupported element dtype {target}")
    h = ctypes.c_void_p()
    dev = get_device() if device is None else int(device)
    code = _lib.DTYPE_F64 if target == np.float64 else _lib.DTYPE_F32
    st = torch_stream(dev) if stream is None else ctypes.c_void_p(int(stream))
    _lib.check(_lib.load().spamm_tree_from_device_on(ctypes.c_void_p(ptr), int(n),
                                                     int(n if ld is None else ld), int(leaf_size),
                                                     code, dev, st, ctypes.byref(h)))
    return _wrap(h.value)


def identity(n, leaf_size=4, dtype=None):
    """Identity matrix as a quadtree (quadtree.py:259-261)."""
    return from_dense(np.eye(n), leaf_size=leaf_size, dtype=dtype)


def to_dense(m, out=None):
    """Function form of m.to_dense() (quadtree.py:264-266)."""
    return m.to_dense(out=out)


def trace(m):
    """Sum of the logical diagonal (quadtree.py:274-277): the diagonal comes
    off the device and numpy's own add.reduce sums it (pairwise order, the
    tree's dtype), so the value is the reference's bit for bit."""
    d = np.empty(m.logical_dim, dtype=m.dtype)
    _lib.check(_lib.load().spamm_tree_diagonal(m._handle, d.ctypes.data_as(ctypes.c_void_p)))
    return float(np.add.reduce(d))


def add(a, b):
    """Tree sum a + b (quadtree.py:280-293): where only one operand has a
    nonzero block that block passes through bit-identically; blocks that
    cancel to zero become Empty."""
    _require_conformable(a, b)
    h = ctypes.c_void_p()
    _lib.check(_lib.load().spamm_tree_add(a._handle, b._handle, ctypes.byref(h)))
    return _wrap(h.value)


def scale(m, s):
    """Tree scaled by a scalar in the tree's dtype (quadtree.py:296-299);
    scaling by 0 yields the Empty tree."""
    h = ctypes.c_void_p()
    _lib.check(_lib.load().spamm_tree_scale(m._handle, float(m.dtype.type(s)), ctypes.byref(h)))
    return _wrap(h.value)


def filter_drop(m, tau):
    """Drop every leaf whose Frobenius norm is < tau (quadtree.py:302-316);
    returns ``m`` itself when nothing drops.  tau < 0 is rejected."""
    if tau < 0:
        raise ValueError(f"tau must be >= 0, got {tau}")
    h = ctypes.c_void_p()
    dropped = ctypes.c_int32(0)
    _lib.check(_lib.load().spamm_tree_filter_drop(m._handle, float(tau), ctypes.byref(h),
                                                  ctypes.byref(dropped)))
    if not dropped.value:
        return m
    return _wrap(h.value)


def tc2_update(x, x2, make_y, rows=None):
    """One TC2 sweep's element-wise work in one device pass (extension;
    spamm_tc2_update in the C ABI): the root squared norms of
    D = add(x2, scale(x, -1)) and, if ``make_y``, of E = add(Y, scale(x, -1)),
    plus Y = add(scale(x, 2), scale(x2, -1)) itself -- bit-identical to those
    tree operations (quadtree.py:280-299), without building D or E.
    ``rows=(lo, hi)`` restricts it to block rows [lo, hi) (a row band).

    Returns (y or None, d, e or None, d_root_nsq, e_root_nsq); d and e are
    norms-only trees (their pyramids; no element storage)."""
    _require_conformable(x, x2)
    lo, hi = (0, x.block_grid) if rows is None else rows
    y, d, e = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    roots = np.zeros(2, np.float64)
    _lib.check(_lib.load().spamm_tc2_update(x._handle, x2._handle, int(bool(make_y)), int(lo),
                                            int(hi), ctypes.byref(y), ctypes.byref(d),
                                            ctypes.byref(e), roots.ctypes.data))
    return (_wrap(y.value) if y.value else None, _wrap(d.value),
            _wrap(e.value) if e.value else None, float(roots[0]), float(roots[1]))


def node_norm(m):
    """Frobenius norm from the root's cached norm (quadtree.py:269-271)."""
    return m.norm()


def audit_norm_cache(m):
    """Maximum relative discrepancy between the cached norm pyramid and one
    recomputed from the leaf data (quadtree.py:325-340); 0.0 for a healthy
    tree.  The recomputation is K1 on the device into scratch storage."""
    nsq = m._pyramid()[2]
    fresh = np.empty_like(nsq)
    _lib.check(_lib.load().spamm_tree_recompute_norms(m._handle, fresh.ctypes.data))
    worst = 0.0
    for off, side in _level_slices(m.depth):
        stored = nsq[off:off + side * side]
        denom = np.where(stored > 0, stored, 1.0)
        worst = max(worst, float((np.abs(fresh[off:off + side * side] - stored) / denom).max()))
    return worst
