"""Host-side behaviour of the drop-in API that needs no GPU: validation and
exception types mirror the reference (quadtree.py:218-251, multiply.py:43-74,
:77-116), and the compute path refuses to run without the CUDA library/GPU
instead of falling back to the CPU."""

import dataclasses
import math

import numpy as np
import pytest

import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import quadtree


def test_config_validation():
    for bad in (-1e-9, float("nan"), float("inf"), -float("inf")):
        with pytest.raises(ValueError):
            sp.SpammConfig(tau=bad)
    cfg = sp.SpammConfig(tau=1e-8)
    assert cfg.count_stats and cfg.deterministic and not cfg.collect_boxes
    with pytest.raises(dataclasses.FrozenInstanceError):
        cfg.tau = 1.0


def test_stats_and_boxes():
    st = sp.ProductStats(leaf_matmuls=3, pruned_volume=10, empty_skip_volume=7)
    assert st.covered_volume(2) == 3 * 8 + 17
    assert st.boxes is None
    bx = sp.PrunedBox(0, 4, 8, 4, 2)
    assert bx == sp.PrunedBox(0, 4, 8, 4, 2)
    assert sp.ProductStats() == sp.ProductStats()


@pytest.mark.parametrize("leaf", [0, 3, 6, -4])
def test_bad_leaf_size(leaf):
    with pytest.raises(ValueError):
        sp.from_dense(np.eye(4), leaf_size=leaf)


def test_bad_dtype():
    with pytest.raises(ValueError):
        sp.from_dense(np.eye(4), dtype=np.int32)
    with pytest.raises(ValueError):
        sp.from_dense(np.eye(4), dtype=np.float16)


def test_non_square_and_empty():
    with pytest.raises(sp.DimensionMismatchError):
        sp.from_dense(np.ones((3, 4)))
    with pytest.raises(sp.DimensionMismatchError):
        sp.from_dense(np.ones(5))
    assert issubclass(sp.DimensionMismatchError, ValueError)
    with pytest.raises(ValueError):
        sp.from_dense(np.zeros((0, 0)))


def test_direct_construction_rejected():
    with pytest.raises(TypeError):
        sp.QuadTreeMatrix()


def test_conformability_checked_in_python():
    class Fake:
        def __init__(self, n, leaf, dtype):
            self.logical_dim, self.leaf_size, self.dtype = n, leaf, np.dtype(dtype)

    with pytest.raises(sp.DimensionMismatchError):
        quadtree._require_conformable(Fake(16, 4, np.float64), Fake(32, 4, np.float64))
    with pytest.raises(sp.DimensionMismatchError):
        quadtree._require_conformable(Fake(16, 4, np.float64), Fake(16, 2, np.float64))
    with pytest.raises(sp.DimensionMismatchError):
        quadtree._require_conformable(Fake(16, 4, np.float64), Fake(16, 4, np.float32))


def test_no_cpu_fallback_without_gpu():
    """On a machine without a CUDA device the product path raises; it never
    computes on the host."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises((RuntimeError, ValueError)):
        sp.from_dense(np.eye(8), leaf_size=4)
    with pytest.raises((RuntimeError, ValueError)):
        sp.from_dense(np.eye(8), leaf_size=4, wait=False)  # the asynchronous build too


def test_public_surface_matches_reference_names():
    ref_hot_path = ["EMPTY", "DimensionMismatchError", "EmptyNode", "InteriorNode", "LeafNode",
                    "QuadTreeMatrix", "from_dense", "identity", "node_norm", "to_dense",
                    "ProductStats", "PrunedBox", "SpammConfig", "exact_multiply",
                    "multiply_error", "spamm"]
    for name in ref_hot_path:
        assert hasattr(sp, name), name
    assert sp.EMPTY.kind == "empty" and sp.EMPTY.norm_sq == 0.0
    assert math.isclose(sp.LeafNode(None, 4.0).norm_sq, 4.0)


def test_async_build_validates_like_from_dense():
    """from_dense(wait=False) validates on the host exactly like the
    synchronous call (reference exception types, before any device work)."""
    with pytest.raises(ValueError):
        sp.from_dense(np.eye(8), leaf_size=3, wait=False)
    with pytest.raises(sp.DimensionMismatchError):
        sp.from_dense(np.ones((4, 5)), leaf_size=4, wait=False)
    with pytest.raises(ValueError):
        sp.from_dense(np.eye(8), leaf_size=4, dtype=np.int32, wait=False)


def test_pending_blocks_wait_is_idempotent_without_a_handle():
    """PendingBlocks.wait() returns its (ids, blocks) and is a no-op once done."""
    from paper_1011_3534_b200.quadtree import PendingBlocks
    ids = np.arange(3)
    blocks = np.zeros((3, 2, 2))
    p = PendingBlocks(None, ids, blocks)
    assert p.wait()[0] is ids and p.wait()[1] is blocks


def test_shim_aliases_every_submodule():
    """The shim maps the reference's module names onto this package's."""
    import sys

    from paper_1011_3534_b200 import compat

    pkg = compat.install()
    try:
        import spamm

        assert spamm is pkg
        for m in compat.SUBMODULES:
            assert sys.modules[f"spamm.{m}"].__name__ == f"paper_1011_3534_b200.{m}"
        from spamm.multiply import SpammConfig, spamm as fn  # noqa: F401
        from spamm.quadtree import from_dense, to_dense  # noqa: F401
    finally:
        compat.uninstall()
    assert "spamm" not in sys.modules or sys.modules["spamm"] is not pkg
