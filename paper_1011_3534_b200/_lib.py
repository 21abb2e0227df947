"""ctypes binding of the C ABI in include/spamm_b200.h.

The CUDA library is the only compute path: if libspamm_b200.so is missing
or no CUDA device is visible, calls raise -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libspamm_b200.so")

SPAMM_OK = 0
SPAMM_ERR_VALUE = 1
SPAMM_ERR_DIMENSION = 2
SPAMM_ERR_CUDA = 3
SPAMM_ERR_NOMEM = 4
SPAMM_ERR_INTERNAL = 5

DTYPE_F64 = 0
DTYPE_F32 = 1

COLLECT_BOXES = 0x1
COUNT_STATS = 0x2
TIER_TAU_DECAY = 0x4
KEEP_TRIPLES = 0x8
TIERED_TRAVERSAL = 0x10
TRAVERSE_ONLY = 0x20
KEEP_PRUNED = 0x40
NEED_BLOCKS = 0x80

# every symbol include/spamm_b200.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "spamm_last_error", "spamm_device_count", "spamm_version",
    "spamm_tree_from_host", "spamm_tree_from_device", "spamm_tree_from_padded_device",
    "spamm_tree_info_get", "spamm_tree_to_host", "spamm_tree_padded_to_host",
    "spamm_tree_pyramid_to_host", "spamm_tree_device_ptrs", "spamm_tree_diff_norm",
    "spamm_tree_free", "spamm_multiply", "spamm_multiply_rows", "spamm_product_boxes",
    "spamm_product_triples", "spamm_product_free",
    "spamm_tree_add", "spamm_tree_scale", "spamm_tree_filter_drop", "spamm_tree_diagonal",
    "spamm_tree_blocks_to_host", "spamm_boxes_morton_order", "spamm_tree_toeplitz",
    "spamm_tree_tridiagonal", "spamm_tree_recompute_norms",
    "spamm_tree_blocks_to_host_async", "spamm_transfer_wait", "spamm_tree_from_host_async",
    "spamm_tree_wait", "spamm_product_pruned", "spamm_product_pruned_count",
    "spamm_tree_band_from_device", "spamm_tree_band_set", "spamm_tree_pyramid_rebuild",
    "spamm_tree_blocks_gather_device", "spamm_tree_blocks_scatter_device",
    "spamm_tree_diagonal_rows", "spamm_tc2_update",
    "spamm_stream_wait", "spamm_stream_signal", "spamm_tree_from_device_on", "spamm_multiply_on",
    "spamm_product_need_blocks",
)


class TreeInfo(ctypes.Structure):
    _fields_ = [("logical_dim", ctypes.c_int64), ("padded_dim", ctypes.c_int64),
                ("block_grid", ctypes.c_int64), ("leaf_size", ctypes.c_int32),
                ("depth", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("device", ctypes.c_int32), ("root_norm_sq", ctypes.c_double)]


class Stats(ctypes.Structure):
    _fields_ = [("leaf_matmuls", ctypes.c_int64), ("pruned_calls", ctypes.c_int64),
                ("pruned_volume", ctypes.c_int64), ("empty_skip_volume", ctypes.c_int64),
                ("max_depth_reached", ctypes.c_int32), ("reserved0", ctypes.c_int32),
                ("omitted_budget", ctypes.c_double), ("n_boxes", ctypes.c_int64),
                ("n_triples", ctypes.c_int64), ("n_groups", ctypes.c_int64),
                ("tier_candidates", ctypes.c_int64 * 32),
                ("tier_survivors", ctypes.c_int64 * 32),
                ("tier_pruned", ctypes.c_int64 * 32),
                ("ms_cull", ctypes.c_float), ("ms_leaf", ctypes.c_float),
                ("ms_ctree", ctypes.c_float), ("ms_total", ctypes.c_float),
                ("ms_gemm", ctypes.c_float), ("kernel_launches", ctypes.c_int32),
                ("traverse_phase_us", ctypes.c_float * 14)]


_lock = threading.Lock()
_lib = None


def load(path=LIB_PATH):
    """Load the library (no CUDA call is made here)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"spamm CUDA library not built: {path} is missing "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
        L = ctypes.CDLL(path)
        vp, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
        pp = ctypes.POINTER(ctypes.c_void_p)
        L.spamm_last_error.restype = ctypes.c_char_p
        L.spamm_version.restype = ctypes.c_char_p
        L.spamm_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
        L.spamm_tree_from_host.argtypes = [vp, i64, i64, i32, i32, i32, pp]
        L.spamm_tree_from_host_async.argtypes = [vp, i64, i64, i32, i32, i32, pp]
        L.spamm_tree_wait.argtypes = [vp]
        L.spamm_tree_from_device.argtypes = [vp, i64, i64, i32, i32, i32, pp]
        L.spamm_tree_from_padded_device.argtypes = [vp, i64, i64, i32, i32, i32, pp]
        L.spamm_tree_info_get.argtypes = [vp, ctypes.POINTER(TreeInfo)]
        L.spamm_tree_to_host.argtypes = [vp, vp, i64]
        L.spamm_tree_padded_to_host.argtypes = [vp, vp]
        L.spamm_tree_pyramid_to_host.argtypes = [vp, vp, vp]
        L.spamm_tree_device_ptrs.argtypes = [vp, pp, pp, pp]
        L.spamm_tree_diff_norm.argtypes = [vp, vp, ctypes.POINTER(ctypes.c_double)]
        L.spamm_tree_add.argtypes = [vp, vp, pp]
        L.spamm_tree_scale.argtypes = [vp, ctypes.c_double, pp]
        L.spamm_tree_filter_drop.argtypes = [vp, ctypes.c_double, pp, ctypes.POINTER(i32)]
        L.spamm_tree_diagonal.argtypes = [vp, vp]
        L.spamm_tree_blocks_to_host.argtypes = [vp, vp, i64, vp]
        L.spamm_tree_blocks_to_host_async.argtypes = [vp, vp, i64, vp, pp]
        L.spamm_transfer_wait.argtypes = [vp]
        L.spamm_tree_free.argtypes = [vp]
        L.spamm_tree_free.restype = None
        L.spamm_multiply.argtypes = [vp, vp, ctypes.c_double, u32, pp, ctypes.POINTER(Stats), pp]
        L.spamm_multiply_on.argtypes = [vp, vp, ctypes.c_double, u32, vp, pp, ctypes.POINTER(Stats),
                                        pp]
        L.spamm_stream_wait.argtypes = [i32, vp]
        L.spamm_stream_signal.argtypes = [i32, vp]
        L.spamm_tree_from_device_on.argtypes = [vp, i64, i64, i32, i32, i32, vp, pp]
        L.spamm_multiply_rows.argtypes = [vp, vp, ctypes.c_double, u32, i64, i64, pp,
                                          ctypes.POINTER(Stats), pp]
        L.spamm_product_boxes.argtypes = [vp, vp, i64]
        L.spamm_product_triples.argtypes = [vp, vp, i64]
        L.spamm_product_free.argtypes = [vp]
        L.spamm_product_free.restype = None
        L.spamm_boxes_morton_order.argtypes = [vp, i64, i32, vp]
        L.spamm_tree_recompute_norms.argtypes = [vp, vp]
        L.spamm_tree_toeplitz.argtypes = [vp, i64, i32, i32, i32, pp]
        L.spamm_tree_tridiagonal.argtypes = [vp, vp, i64, i32, i32, i32, pp]
        L.spamm_product_pruned.argtypes = [vp, vp, vp, i64]
        L.spamm_product_pruned_count.argtypes = [vp]
        L.spamm_product_pruned_count.restype = i64
        L.spamm_product_need_blocks.argtypes = [vp, vp, i64]
        L.spamm_tree_band_from_device.argtypes = [vp, i64, i64, i32, i32, i64, i64, i32, pp]
        L.spamm_tree_band_set.argtypes = [vp, i64, i64]
        L.spamm_tree_pyramid_rebuild.argtypes = [vp]
        L.spamm_tree_blocks_gather_device.argtypes = [vp, vp, i64, vp]
        L.spamm_tree_blocks_scatter_device.argtypes = [vp, vp, i64, vp]
        L.spamm_tree_diagonal_rows.argtypes = [vp, i64, i64, vp]
        L.spamm_tc2_update.argtypes = [vp, vp, i32, i64, i64, pp, pp, pp, vp]
        _lib = L
        return L


def check(rc):
    """Map a C status code to the reference's exception types."""
    if rc == SPAMM_OK:
        return
    msg = load().spamm_last_error().decode(errors="replace")
    if rc == SPAMM_ERR_DIMENSION:
        from .quadtree import DimensionMismatchError
        raise DimensionMismatchError(msg)
    if rc == SPAMM_ERR_VALUE:
        raise ValueError(msg)
    if rc == SPAMM_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"spamm_b200: {msg}")


def device_count():
    n = ctypes.c_int(0)
    check(load().spamm_device_count(ctypes.byref(n)))
    return n.value
