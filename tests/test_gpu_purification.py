"""Tree algebra and the TC2 purification driver on the GPU vs the reference
(tests/golden/purify_golden.*, produced by the real reference package):
add / scale / filter_drop results bit for bit (padded arrays and pyramids),
traces exactly, and purify() reproducing the reference's final density, trace
history, per-sweep leaf multiplies and energies on a 1-D chain (SpAMM and
dropping modes) and on the 3-D Morton-ordered lattice of BASELINE config 4."""

import json
import os

import numpy as np
import pytest

import paper_1011_3534_b200 as sp
from paper_1011_3534_b200 import purification as P

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def golden():
    z = np.load(os.path.join(HERE, "purify_golden.npz"))
    with open(os.path.join(HERE, "purify_golden.json")) as fh:
        meta = json.load(fh)
    return z, meta


def _same_tree(t, z, prefix):
    pad = z[prefix + "_padded"]
    got = t._padded
    assert got.dtype == pad.dtype
    assert np.array_equal(got.view(np.uint8), pad.view(np.uint8)), prefix + " padded"
    nsq, occ = t._pyramid()[2], t._pyramid()[3]
    assert np.array_equal(nsq.view(np.uint64), z[prefix + "_nsq"].view(np.uint64)), prefix + " nsq"
    assert np.array_equal(occ, z[prefix + "_occ"]), prefix + " occ"


@pytest.mark.parametrize("dname", ["f64", "f32"])
def test_algebra_bit_exact(golden, dname):
    z, meta = golden
    a, b = z[f"{dname}_a"], z[f"{dname}_b"]
    ta = sp.from_dense(a, leaf_size=8, dtype=a.dtype)
    tb = sp.from_dense(b, leaf_size=8, dtype=b.dtype)
    _same_tree(sp.add(ta, tb), z, f"{dname}_add")
    _same_tree(sp.scale(ta, -1.5), z, f"{dname}_scale_m15")
    _same_tree(sp.scale(ta, 0.0), z, f"{dname}_scale_0")
    _same_tree(sp.scale(tb, 1.0 / 3.0), z, f"{dname}_scale_third")
    _same_tree(sp.filter_drop(ta, meta[f"{dname}_tau_mid"]), z, f"{dname}_filter_mid")
    assert (sp.filter_drop(ta, 0.0) is ta) == meta[f"{dname}_filter_none_is_input"]
    assert sp.trace(ta) == meta[f"{dname}_trace_a"]
    assert sp.trace(sp.add(ta, tb)) == meta[f"{dname}_trace_add"]


def test_algebra_errors():
    t = sp.from_dense(np.eye(8), leaf_size=4)
    u = sp.from_dense(np.eye(16), leaf_size=4)
    with pytest.raises(sp.DimensionMismatchError):
        sp.add(t, u)
    with pytest.raises(ValueError):
        sp.filter_drop(t, -1.0)


@pytest.mark.parametrize("case", ["chain64_spamm", "chain64_drop", "lattice4_spamm",
                                  "lattice8_spamm"])
def test_purify_matches_reference(golden, case):
    z, meta = golden
    m = meta[case]
    f = sp.from_dense(z[f"{case}_f"], leaf_size=m["leaf"])
    mode = (P.SpammMode if m["mode"] == "SpammMode" else P.DroppingMode)(m["tau"])
    res = P.purify(f, m["n_occ"], mode, max_iter=m["max_iter"])
    assert res.step_leaf_matmuls == m["step_leaf_matmuls"]
    assert res.total_leaf_matmuls == m["total_leaf_matmuls"]
    assert res.trace_history == m["trace_history"]
    assert np.array_equal(res.density._padded.view(np.uint64),
                          z[f"{case}_density"].view(np.uint64)), "density"
    assert res.energy == m["energy"]
    assert res.reference_energy == m["reference_energy"]
    assert res.delta_e_rel == m["delta_e_rel"]


def test_purify_validation():
    f = sp.from_dense(np.diag([-1.0, 1.0]), leaf_size=1)
    with pytest.raises(ValueError):
        P.purify(f, 1, P.SpammMode(1e-8), max_iter=0)
    with pytest.raises(ValueError):
        P.purify(f, 1, P.SpammMode(-1.0))
    with pytest.raises(ValueError):
        P.purify(f, 3, P.SpammMode(1e-8))
    with pytest.raises(ValueError):
        P.purify(sp.from_dense(np.array([[0.0, 1.0], [2.0, 0.0]]), leaf_size=1), 1,
                 P.SpammMode(1e-8))
    with pytest.raises(TypeError):
        P.tc2_step(f, 1, object())


def test_purify_two_level_analytic():
    f = sp.from_dense(np.diag([-1.0, 1.0]))
    for mode in (P.SpammMode(0.0), P.SpammMode(1e-8), P.DroppingMode(1e-8)):
        res = P.purify(f, 1, mode)
        assert np.array_equal(res.density.to_dense(), np.diag([1.0, 0.0]))
        assert res.energy == -1.0
        assert res.delta_e_rel == 0.0


def test_match_error_threshold_boundary(golden):
    z, meta = golden
    f = sp.from_dense(z["chain64_spamm_f"], leaf_size=4)
    res = P.match_error_threshold(f, 32, 1e3, P.SpammMode(0.0))
    assert res.hit_boundary and not res.converged and res.tau == 1e-1
