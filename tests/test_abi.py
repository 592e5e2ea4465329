"""The C-ABI library loads and exports every symbol include/thetis.h declares
(CPU-only: no compute calls), and host-side validation answers without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "thetis.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"THETIS_API\s+[\w\s\*]+?\b(thetis_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for required in ("thetis_build_lp", "thetis_build_graph_lp", "thetis_solve", "thetis_round",
                     "thetis_objective", "thetis_free", "thetis_error_string"):
        assert required in names


def test_library_exports_every_declared_symbol():
    import paper_1311_2661_b200 as th
    lib = ctypes.CDLL(th.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    # the binding wraps exactly the declared boundary
    assert sorted(th.EXPORTED) == declared_symbols()
    out = subprocess.run(["nm", "-D", "--defined-only", th.LIB_PATH], capture_output=True, text=True).stdout
    exported = sorted(set(re.findall(r"\bT (thetis_\w+)", out)))
    assert exported == declared_symbols()


def test_error_strings_and_validation_without_gpu():
    import paper_1311_2661_b200 as th
    assert th.thetis_error_string(0) == b"THETIS_OK"
    assert th.thetis_error_string(-2) == b"THETIS_ERR_WORKSPACE_TOO_SMALL"
    assert th.thetis_version().startswith(b"thetis-b200")
    sz = ctypes.c_size_t()
    assert th.thetis_build_graph_lp_workspace(7, 10, 10, 0, ctypes.byref(sz)) == th.THETIS_ERR_INVALID_ARG
    assert th.thetis_build_graph_lp_workspace(3, 10, 10, 1, ctypes.byref(sz)) == th.THETIS_ERR_INVALID_ARG
    assert th.thetis_build_lp_workspace(-1, 1, 1, ctypes.byref(sz)) == th.THETIS_ERR_INVALID_ARG
    h = ctypes.c_void_p()
    assert th.thetis_build_graph_lp(None, None, 0, None, 1, 1, 0, None, None, None, None, 0, None, 0) == \
        th.THETIS_ERR_INVALID_ARG
    assert th.thetis_solve(None, 1.0, 1, 0, 0, 0, None) == th.THETIS_ERR_INVALID_ARG


def test_kernels_are_sm100a():
    import paper_1311_2661_b200 as th
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", th.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_product_never_references_the_oracle():
    # the product path neither imports nor links anything under oracle/
    pkg = os.path.join(ROOT, "paper_1311_2661_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", text, re.M), f
                assert "thetis_ref" not in text and "libthetis_ref" not in text, f
    out = subprocess.run(["ldd", os.path.join(pkg, "libthetis.so")], capture_output=True, text=True).stdout
    assert "thetis_ref" not in out
