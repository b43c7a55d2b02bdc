"""The C-ABI boundary: libttk.so loads and exports every entry point include/ttk.h declares
(no compute calls; runs without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ttk.h")
LIB = os.path.join(ROOT, "paper_1906_06785_b200", "libttk.so")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tk_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def so():
    if not os.path.exists(LIB):
        from paper_1906_06785_b200.build import build
        build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ["tk_apply_op", "tk_round", "tk_dot", "tk_axpby", "tk_norm", "tk_op_create",
              "tk_ctx_create", "tk_gmres_cycle"]:
        assert s in syms


def test_library_exports_every_declared_symbol(so):
    missing = [s for s in declared_symbols() if not hasattr(so, s)]
    assert not missing, missing


def test_binding_names_match_header():
    from paper_1906_06785_b200 import ttk
    assert sorted(ttk.EXPORTED) == declared_symbols()


def test_version_string(so):
    so.tk_version.restype = ctypes.c_char_p
    assert b"sm_100a" in so.tk_version()


def test_null_context_is_rejected(so):
    # argument validation happens before any CUDA call
    assert so.tk_ctx_create(None, None) == -3


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1906_06785_b200")
    pat = re.compile(r"^\s*(from\s+oracle|import\s+oracle)|oracle/", re.M)
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                assert not pat.search(open(os.path.join(dirpath, f)).read()), f


def test_new_entry_points_reject_null_arguments(so):
    """tk_op_group_space / tk_gmres_solve validate their arguments before any CUDA call."""
    so.tk_op_group_space.argtypes = [ctypes.c_void_p, ctypes.c_int]
    assert so.tk_op_group_space(None, 1) == -3
    so.tk_gmres_solve.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 2 + \
        [ctypes.c_double] * 3 + [ctypes.c_void_p] * 5
    assert so.tk_gmres_solve(None, None, None, 4, 2, 1e-8, 1e-6, -1.0, None, None, None, None,
                             None) == -3
