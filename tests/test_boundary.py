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


def test_round2_entry_points_reject_null_arguments(so):
    """NEXT-3 / NEXT-4 / async entry points validate their handles before any CUDA call."""
    P = ctypes.c_void_p
    so.tk_sync_ranks.argtypes = [P, P]
    assert so.tk_sync_ranks(None, None) == -3
    so.tk_ctx_set_async.argtypes = [P, ctypes.c_int]
    assert so.tk_ctx_set_async(None, 1) == -3
    so.tk_prec_apply.argtypes = [P, P, ctypes.c_int, P, P]
    assert so.tk_prec_apply(None, None, 0, None, None) == -3
    so.tk_bt_solve.argtypes = [P, P, P, ctypes.c_int64, ctypes.c_int, P]
    assert so.tk_bt_solve(None, None, None, 0, 1, None) == -3
    so.tk_picard.argtypes = [P] * 5 + [ctypes.c_double, ctypes.c_int] + [ctypes.c_double] * 3 + \
        [ctypes.c_int] * 2 + [P] * 4
    assert so.tk_picard(None, None, None, None, None, 1e-3, 5, 0.1, 1e-3, -1.0, 10, 3, None, None,
                        None, None) == -3
    so.tk_prec_operator.argtypes = [P, ctypes.c_int]
    so.tk_prec_operator.restype = P
    assert so.tk_prec_operator(None, 0) is None


def test_round_workspace_bound_is_a_host_function(so):
    """tk_round_workspace_bytes is pure host arithmetic: callable without a GPU, zero for
    invalid sizes, monotone in every argument, and >= the caller-owned-free minimum (the
    grown space core's Gram pass needs at least n_x * min(R1, n_xi * min(n_t, R2)) doubles)."""
    f = so.tk_round_workspace_bytes
    f.argtypes = [ctypes.c_int64] * 5
    f.restype = ctypes.c_size_t
    assert f(0, 1, 1, 1, 1) == 0 and f(10, 1, 1, 1, -1) == 0
    base = (12288, 35, 64, 120, 120)
    b0 = f(*base)
    assert b0 >= 8 * 12288 * min(120, 35 * 64)
    for i in range(5):
        bigger = list(base)
        bigger[i] *= 2
        assert f(*bigger) >= b0
    # c4 grown ranks: a few GB of scratch, far inside 180 GB of HBM
    c4 = f(786432, 165, 512, 896, 896)
    assert 4e9 < c4 < 3e10


def test_gemm_and_schedule_entry_points_reject_null_arguments(so):
    """tk_gemm / tk_ctx_set_gemm_feed / tk_ctx_set_jacobi_schedule validate their handles before
    any CUDA call (no GPU needed)."""
    P, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    so.tk_gemm.argtypes = [P, I, I, I64, I64, I64, D, P, I64, P, I64, D, P, I64, I]
    assert so.tk_gemm(None, 0, 0, 4, 4, 4, 1.0, None, 4, None, 4, 0.0, None, 4, 0) == -3
    so.tk_ctx_set_gemm_feed.argtypes = [P, I]
    assert so.tk_ctx_set_gemm_feed(None, 1) == -3
    so.tk_ctx_set_jacobi_schedule.argtypes = [P, I]
    assert so.tk_ctx_set_jacobi_schedule(None, 1) == -3
    so.tk_ctx_gate_stream.argtypes = [P, P]
    assert so.tk_ctx_gate_stream(None, None) == -3
