"""The C ABI library: it loads without a GPU and exports exactly the entry
points include/spamm_b200.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_1011_3534_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spamm_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"SPAMM_API[^;]*?\b(spamm_\w+)\s*\(", text, re.S)))


def test_header_declares_entry_points():
    names = declared()
    assert "spamm_multiply" in names and "spamm_tree_from_host" in names
    assert sorted(_lib.EXPORTED) == names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("CUDA library not built (run __graft_entry__.build())")
    out = subprocess.check_output(["nm", "-D", "--defined-only", _lib.LIB_PATH]).decode()
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    # nothing but the C ABI is exported
    assert all(n.startswith("spamm_") for n in exported), sorted(exported)
    L = _lib.load()
    for n in declared():
        assert isinstance(getattr(L, n), ctypes._CFuncPtr)


def test_version_string():
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("CUDA library not built")
    assert _lib.load().spamm_version().decode().startswith("spamm_b200")


def test_structs_match_header_sizes():
    # spamm_stats / spamm_tree_info layouts mirrored in ctypes
    text = open(HEADER).read()
    assert "float traverse_phase_us[14];" in text
    assert ctypes.sizeof(_lib.TreeInfo) == 8 * 3 + 4 * 4 + 8
    assert ctypes.sizeof(_lib.Stats) % 8 == 0
