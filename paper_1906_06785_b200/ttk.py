"""Thin ctypes binding of libttk (include/ttk.h).  Argument marshalling only: every step of
the path runs in the library's CUDA kernels; there is no CPU fallback.  PyTorch provides
device memory (the caller-owned TT core buffers) and the CUDA stream.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libttk.so")

TK_OK, TK_ESHAPE, TK_ECAP, TK_EARG, TK_ENUMERIC, TK_ECUDA = 0, -1, -2, -3, -4, -5
_CODES = {TK_ESHAPE: "TK_ESHAPE", TK_ECAP: "TK_ECAP", TK_EARG: "TK_EARG",
          TK_ENUMERIC: "TK_ENUMERIC", TK_ECUDA: "TK_ECUDA"}

EXPORTED = ["tk_version", "tk_ctx_create", "tk_ctx_destroy", "tk_last_error", "tk_ctx_launch_count",
            "tk_ctx_profile", "tk_ctx_profile_dump",
            "tk_op_create", "tk_op_destroy", "tk_op_terms", "tk_apply_op", "tk_round",
            "tk_apply_round", "tk_dot",
            "tk_norm", "tk_axpby", "tk_axpby_host", "tk_scale", "tk_gmres_cycle",
            "tk_gmres_solve", "tk_op_group_space", "tk_op_set_spmm_kernel", "tk_op_concat",
            "tk_conv_create", "tk_conv_destroy", "tk_op_convection",
            "tk_bt_create", "tk_bt_create_gram", "tk_bt_destroy", "tk_bt_solve",
            "tk_prec_create_lsc", "tk_prec_destroy", "tk_prec_apply", "tk_prec_operator",
            "tk_gmres_cycle_p", "tk_gmres_solve_p", "tk_picard",
            "tk_ctx_set_async", "tk_sync_ranks", "tk_round_workspace_bytes", "tk_ctx_reserve",
            "tk_ctx_scratch_high_water", "tk_gemm", "tk_ctx_set_gemm_feed",
            "tk_ctx_set_jacobi_schedule", "tk_ctx_gate_stream"]


class TkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_CODES.get(code, code)}: {msg}")
        self.code = code


class tk_tt(ctypes.Structure):
    _fields_ = [("n_x", ctypes.c_int64), ("n_xi", ctypes.c_int64), ("n_t", ctypes.c_int64),
                ("r1", ctypes.c_int64), ("r2", ctypes.c_int64),
                ("cap1", ctypes.c_int64), ("cap2", ctypes.c_int64),
                ("U1", ctypes.c_void_p), ("U2", ctypes.c_void_p), ("U3", ctypes.c_void_p)]


_lib = None


def lib():
    """Load libttk.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"libttk.so not built at {_LIB_PATH}; run __graft_entry__.build()")
    L = ctypes.CDLL(_LIB_PATH)
    P, I64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    PP = ctypes.POINTER(ctypes.c_void_p)
    L.tk_version.restype = ctypes.c_char_p
    L.tk_ctx_create.argtypes = [ctypes.POINTER(P), P]
    L.tk_ctx_destroy.argtypes = [P]
    L.tk_last_error.argtypes = [P]
    L.tk_last_error.restype = ctypes.c_char_p
    L.tk_ctx_launch_count.argtypes = [P]
    L.tk_ctx_launch_count.restype = I64
    L.tk_op_create.argtypes = [P, ctypes.POINTER(P), I, I64, I64, I64, PP, PP, PP, PP,
                               ctypes.POINTER(I), ctypes.POINTER(I), PP]
    L.tk_op_destroy.argtypes = [P]
    L.tk_op_terms.argtypes = [P]
    L.tk_op_group_space.argtypes = [P, I]
    L.tk_op_set_spmm_kernel.argtypes = [P, I]
    TTP = ctypes.POINTER(tk_tt)
    L.tk_op_concat.argtypes = [P, I, PP, ctypes.POINTER(P)]
    L.tk_conv_create.argtypes = [P, ctypes.POINTER(P), I64, I64, I64, I, I64, PP, PP, PP, P]
    L.tk_conv_destroy.argtypes = [P]
    L.tk_op_convection.argtypes = [P, P, TTP, ctypes.POINTER(P)]
    DP = ctypes.POINTER(D)
    L.tk_apply_op.argtypes = [P, P, TTP, TTP]
    L.tk_round.argtypes = [P, TTP, D, I64, DP, DP, DP, DP]
    L.tk_apply_round.argtypes = [P, P, TTP, TTP, D, I64, DP, DP, DP, DP]
    L.tk_dot.argtypes = [P, TTP, TTP, P]
    L.tk_norm.argtypes = [P, TTP, P]
    L.tk_axpby.argtypes = [P, P, TTP, P, TTP, TTP]
    L.tk_axpby_host.argtypes = [P, D, TTP, D, TTP, TTP]
    L.tk_scale.argtypes = [P, TTP, P, I]
    L.tk_gmres_cycle.argtypes = [P, P, TTP, I, D, DP, ctypes.POINTER(I), DP, DP]
    L.tk_gmres_solve.argtypes = [P, P, TTP, I, I, D, D, D, TTP, DP, DP, ctypes.POINTER(I),
                                 ctypes.POINTER(I)]
    IP = ctypes.POINTER(ctypes.c_int32)
    L.tk_bt_create.argtypes = [P, ctypes.POINTER(P), I64, I64, P, P, P, D]
    L.tk_bt_create_gram.argtypes = [P, ctypes.POINTER(P), I64, I64, I64, P, P, P]
    L.tk_bt_destroy.argtypes = [P]
    L.tk_bt_solve.argtypes = [P, P, TTP, I64, I, TTP]
    L.tk_prec_create_lsc.argtypes = [P, ctypes.POINTER(P), I64, I64, I64, P, P, P, P, P, P, D, D,
                                     D, I, I]
    L.tk_prec_destroy.argtypes = [P]
    L.tk_prec_apply.argtypes = [P, P, I, TTP, TTP]
    L.tk_prec_operator.argtypes = [P, I]
    L.tk_prec_operator.restype = P
    L.tk_gmres_cycle_p.argtypes = [P, P, P, TTP, I, D, DP, ctypes.POINTER(I), DP, DP]
    L.tk_gmres_solve_p.argtypes = [P, P, P, TTP, I, I, D, D, D, TTP, DP, DP, ctypes.POINTER(I),
                                   ctypes.POINTER(I)]
    L.tk_picard.argtypes = [P, P, P, P, TTP, D, I, D, D, D, I, I, TTP, DP, ctypes.POINTER(I),
                            ctypes.POINTER(I64)]
    L.tk_ctx_set_async.argtypes = [P, I]
    L.tk_sync_ranks.argtypes = [P, TTP]
    L.tk_round_workspace_bytes.argtypes = [I64, I64, I64, I64, I64]
    L.tk_round_workspace_bytes.restype = ctypes.c_size_t
    L.tk_ctx_reserve.argtypes = [P, ctypes.c_size_t]
    L.tk_ctx_scratch_high_water.argtypes = [P, I]
    L.tk_ctx_scratch_high_water.restype = I64
    L.tk_gemm.argtypes = [P, I, I, I64, I64, I64, D, P, I64, P, I64, D, P, I64, I]
    L.tk_ctx_set_gemm_feed.argtypes = [P, I]
    L.tk_ctx_set_jacobi_schedule.argtypes = [P, I]
    L.tk_ctx_gate_stream.argtypes = [P, P]
    L.tk_ctx_profile.argtypes = [P, I]
    L.tk_ctx_profile_dump.argtypes = [P, ctypes.c_char_p, ctypes.c_size_t]
    for name in EXPORTED:
        if name not in ("tk_version", "tk_last_error", "tk_ctx_launch_count",
                        "tk_prec_operator", "tk_round_workspace_bytes",
                        "tk_ctx_scratch_high_water"):
            getattr(L, name).restype = I
    _lib = L
    return L


def _require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1906_06785_b200 needs a CUDA device (B200); no CPU fallback")


class Context:
    """A libttk context bound to the current torch CUDA stream."""

    def __init__(self, stream: torch.cuda.Stream | None = None):
        _require_cuda()
        self.stream = stream or torch.cuda.current_stream()
        self._h = ctypes.c_void_p()
        self.async_on = False
        self._pending = []  # (TT, tk_tt struct) of queued async roundings
        rc = lib().tk_ctx_create(ctypes.byref(self._h), ctypes.c_void_p(self.stream.cuda_stream))
        if rc != TK_OK:
            raise TkError(rc, "tk_ctx_create failed")

    def set_async(self, on: bool = True) -> bool:
        """tk_ctx_set_async: queue tk_round / tk_apply_round to the context's worker; the TTs'
        ranks are valid after sync().  Returns whether async mode is on."""
        if not on:
            self.sync()
        rc = lib().tk_ctx_set_async(self._h, 1 if on else 0)
        if rc < 0:
            raise TkError(rc, lib().tk_last_error(self._h).decode())
        self.async_on = bool(on) and rc == 1
        return self.async_on

    def sync(self):
        """tk_sync_ranks: wait for the queued roundings and publish their ranks."""
        pend, self._pending = self._pending, []
        rc = lib().tk_sync_ranks(self._h, None) if self._h else TK_OK
        for t, st in pend:
            if t is not None:
                t._update(st)
        self.check(rc)

    def set_gemm_feed(self, mode: int):
        """0 = cp.async, 1 = TMA tensor tiles (default) for the heavy DMMA products."""
        self.check(lib().tk_ctx_set_gemm_feed(self._h, int(mode)))

    def gate_stream(self, stream: torch.cuda.Stream) -> bool:
        """Work enqueued on `stream` from now on waits (on the device) until the most recently
        submitted rounding of this context has reached its DMMA-bound phase
        (tk_ctx_gate_stream): the window for pipelined bulk copies.  Returns False when the
        driver cannot gate (the stream then runs at once)."""
        rc = lib().tk_ctx_gate_stream(self._h, ctypes.c_void_p(stream.cuda_stream))
        if rc < 0:
            self.check(rc)
        return rc == 1

    def set_jacobi_schedule(self, mode: int):
        """1 = dataflow (default), 0 = grid barriers for the block-Jacobi eigensolver."""
        self.check(lib().tk_ctx_set_jacobi_schedule(self._h, int(mode)))

    def gemm(self, A: torch.Tensor, B: torch.Tensor, C: torch.Tensor, M: int, N: int, K: int,
             trans_a: bool = False, trans_b: bool = False, alpha: float = 1.0, beta: float = 0.0,
             lda: int | None = None, ldb: int | None = None, ldc: int | None = None,
             sym: bool = False):
        """C = alpha op(A) op(B) + beta C on device fp64 buffers (tk_gemm; marshalling only)."""
        lda = lda if lda is not None else (M if trans_a else K)
        ldb = ldb if ldb is not None else (K if trans_b else N)
        ldc = ldc if ldc is not None else N
        self.check(lib().tk_gemm(self._h, int(trans_a), int(trans_b), M, N, K, float(alpha),
                                 A.data_ptr(), lda, B.data_ptr(), ldb, float(beta), C.data_ptr(),
                                 ldc, int(sym)))

    def reserve(self, nbytes: int):
        self.check(lib().tk_ctx_reserve(self._h, int(nbytes)))

    def scratch_high_water(self, reset: bool = False) -> int:
        return int(lib().tk_ctx_scratch_high_water(self._h, 1 if reset else 0))

    def check(self, rc: int):
        if rc != TK_OK:
            raise TkError(rc, lib().tk_last_error(self._h).decode())

    @property
    def launches(self) -> int:
        return int(lib().tk_ctx_launch_count(self._h))

    def close(self):
        """tk_ctx_destroy now (drains the async queue, releases an unused copy-window gate)."""
        if self._h:
            h, self._h = self._h, None
            lib().tk_ctx_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context()
    return _default_ctx


class TT:
    """A 3-core tensor train in caller-owned device buffers (layouts of include/ttk.h)."""

    def __init__(self, n_x, n_xi, n_t, r1, r2, cap1=None, cap2=None, device="cuda"):
        self.n_x, self.n_xi, self.n_t = int(n_x), int(n_xi), int(n_t)
        self._pend = None  # (Context, tk_tt) while an async rounding of this TT is queued
        self._r1, self._r2 = int(r1), int(r2)
        self.cap1 = int(cap1 if cap1 is not None else r1)
        self.cap2 = int(cap2 if cap2 is not None else r2)
        dt = torch.float64
        self.b1 = torch.empty(self.n_x * self.cap1, dtype=dt, device=device)
        self.b2 = torch.empty(self.cap1 * self.n_xi * self.cap2, dtype=dt, device=device)
        self.b3 = torch.empty(self.cap2 * self.n_t, dtype=dt, device=device)

    @classmethod
    def from_cores(cls, u1, u2, u3, cap1=None, cap2=None, non_blocking=False):
        n_x, r1 = u1.shape
        _, n_xi, r2 = u2.shape
        n_t = u3.shape[1]
        t = cls(n_x, n_xi, n_t, r1, r2, cap1, cap2)
        for buf, src in ((t.b1, u1), (t.b2, u2), (t.b3, u3)):
            src_t = torch.as_tensor(np.ascontiguousarray(src) if isinstance(src, np.ndarray) else src,
                                    dtype=torch.float64)
            buf[: src_t.numel()].copy_(src_t.reshape(-1), non_blocking=non_blocking)
        return t

    # ranks: reading them waits for a queued asynchronous rounding of this TT (tk_sync_ranks)
    @property
    def r1(self):
        if self._pend is not None:
            self._pend[0].sync()
        return self._r1

    @property
    def r2(self):
        if self._pend is not None:
            self._pend[0].sync()
        return self._r2

    @property
    def U1(self):
        return self.b1[: self.n_x * self.r1].view(self.n_x, self.r1)

    @property
    def U2(self):
        return self.b2[: self.r1 * self.n_xi * self.r2].view(self.r1, self.n_xi, self.r2)

    @property
    def U3(self):
        return self.b3[: self.r2 * self.n_t].view(self.r2, self.n_t)

    @property
    def ranks(self):
        return self.r1, self.r2

    def cores_numpy(self):
        return (self.U1.cpu().numpy().copy(), self.U2.cpu().numpy().copy(),
                self.U3.cpu().numpy().copy())

    def struct(self) -> tk_tt:
        if self._pend is not None:  # queued: later queued calls share the struct the worker
            return self._pend[1]    # publishes into
        return tk_tt(self.n_x, self.n_xi, self.n_t, self._r1, self._r2, self.cap1, self.cap2,
                     self.b1.data_ptr(), self.b2.data_ptr(), self.b3.data_ptr())

    def _update(self, s: tk_tt):
        self._pend = None
        self._r1, self._r2 = int(s.r1), int(s.r2)

    def _queue(self, ctx, s: tk_tt):
        self._pend = (ctx, s)
        ctx._pending.append((self, s))


class Operator:
    """Device copy of A = sum_k T_k (x) G_k (x) K_k (tk_op_create).

    `terms` is any sequence of objects with attributes K (CSR with indptr/indices/data),
    G (n_xi x n_xi array), kl, ku, band ((kl+ku+1) x n_t LAPACK band array)."""

    def __init__(self, n_x, n_xi, n_t, terms, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.n_x, self.n_xi, self.n_t = int(n_x), int(n_xi), int(n_t)
        T = len(terms)
        self.T = T
        keep = []
        rp, cl, vl, gg, bd = [(ctypes.c_void_p * T)() for _ in range(5)]
        kl = (ctypes.c_int * T)()
        ku = (ctypes.c_int * T)()
        for k, t in enumerate(terms):
            a_rp = np.ascontiguousarray(t.K.indptr, dtype=np.int32)
            a_cl = np.ascontiguousarray(t.K.indices, dtype=np.int32)
            a_vl = np.ascontiguousarray(t.K.data, dtype=np.float64)
            a_g = np.ascontiguousarray(t.G, dtype=np.float64)
            # LAPACK band storage is column-major: element (row, col) at col*ldab + row
            a_b = np.asfortranarray(np.asarray(t.band, dtype=np.float64)).ravel(order="F")
            keep += [a_rp, a_cl, a_vl, a_g, a_b]
            rp[k], cl[k], vl[k] = a_rp.ctypes.data, a_cl.ctypes.data, a_vl.ctypes.data
            gg[k], bd[k] = a_g.ctypes.data, a_b.ctypes.data
            kl[k], ku[k] = int(t.kl), int(t.ku)
        self._h = ctypes.c_void_p()
        self.ctx.check(lib().tk_op_create(self.ctx._h, ctypes.byref(self._h), T, self.n_x,
                                          self.n_xi, self.n_t, rp, cl, vl, gg, kl, ku, bd))

    @classmethod
    def from_kronsum(cls, op, ctx=None):
        return cls(op.n_x, op.n_xi, op.n_t, op.terms, ctx)

    @classmethod
    def _from_handle(cls, h, n_x, n_xi, n_t, ctx) -> "Operator":
        self = cls.__new__(cls)
        self.ctx = ctx
        self.n_x, self.n_xi, self.n_t = int(n_x), int(n_xi), int(n_t)
        self._h = h
        self.T = int(lib().tk_op_terms(h))
        return self

    @classmethod
    def concat(cls, ops) -> "Operator":
        """A = sum_i A_i: the terms of ops[0], ops[1], ... (tk_op_concat)."""
        ctx = ops[0].ctx
        arr = (ctypes.c_void_p * len(ops))(*[o._h.value for o in ops])
        h = ctypes.c_void_p()
        ctx.check(lib().tk_op_concat(ctx._h, len(ops), arr, ctypes.byref(h)))
        o = ops[0]
        return cls._from_handle(h, o.n_x, o.n_xi, o.n_t, ctx)

    def group_space(self, enable: bool = True) -> int:
        """Opt-in exact factor grouping of the space core in tt_apply_round
        (tk_op_group_space); returns the number of spatial groups G (T: nothing groups)."""
        g = lib().tk_op_group_space(self._h, 1 if enable else 0)
        if g < 0:
            raise TkError(g, "tk_op_group_space")
        return g

    def set_spmm_kernel(self, kernel: int) -> bool:
        """Row a1's SpMM kernel (tk_op_set_spmm_kernel): 0 = column-merged multi-term sweep
        (default), 1 = per-term CSR kernel.  Returns True if the merged kernel will run."""
        rc = lib().tk_op_set_spmm_kernel(self._h, int(kernel))
        if rc < 0:
            raise TkError(rc, "tk_op_set_spmm_kernel")
        return rc == 1

    def __del__(self):
        try:
            if self._h:
                lib().tk_op_destroy(self._h)
        except Exception:
            pass


class Convection:
    """The discretisation of the TT convection operator N(u) of eq:N_kron (tk_conv_create):
    d velocity components of n_v dofs at the start of the spatial mode, the n_v x n_v
    difference operators D_c (scipy CSR) of the convective derivative, and the chaos triple
    products H (n_xi x n_xi x n_xi, H[l, r, s] = <psi_l psi_r psi_s>).  operator(u) builds
    N(u) on the device from the velocity TT u (tk_op_convection)."""

    def __init__(self, n_x, n_xi, n_t, D, n_v, H, ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.n_x, self.n_xi, self.n_t = int(n_x), int(n_xi), int(n_t)
        d = len(D)
        rp, cl, vl = [(ctypes.c_void_p * d)() for _ in range(3)]
        keep = []
        for c, m in enumerate(D):
            a_rp = np.ascontiguousarray(m.indptr, dtype=np.int32)
            a_cl = np.ascontiguousarray(m.indices, dtype=np.int32)
            a_vl = np.ascontiguousarray(m.data, dtype=np.float64)
            keep += [a_rp, a_cl, a_vl]
            rp[c], cl[c], vl[c] = a_rp.ctypes.data, a_cl.ctypes.data, a_vl.ctypes.data
        h = np.ascontiguousarray(np.asarray(H, dtype=np.float64).reshape(-1))
        assert h.size == self.n_xi ** 3
        self._h = ctypes.c_void_p()
        self.ctx.check(lib().tk_conv_create(self.ctx._h, ctypes.byref(self._h), self.n_x,
                                            self.n_xi, self.n_t, d, int(n_v), rp, cl, vl,
                                            h.ctypes.data))

    def operator(self, u: "TT") -> Operator:
        us = u.struct()
        h = ctypes.c_void_p()
        self.ctx.check(lib().tk_op_convection(self.ctx._h, self._h, ctypes.byref(us),
                                              ctypes.byref(h)))
        return Operator._from_handle(h, self.n_x, self.n_xi, self.n_t, self.ctx)

    def __del__(self):
        try:
            if self._h:
                lib().tk_conv_destroy(self._h)
        except Exception:
            pass


# ----------------------------------------------------------------------------- the path
def tt_apply_op(op: Operator, x: TT, out: TT | None = None) -> TT:
    """y = A x (tk_apply_op); y ranks (T r1, T r2)."""
    ctx = op.ctx
    y = out or TT(x.n_x, x.n_xi, x.n_t, op.T * x.r1, op.T * x.r2)
    xs, ys = x.struct(), y.struct()
    ctx.check(lib().tk_apply_op(ctx._h, op._h, ctypes.byref(xs), ctypes.byref(ys)))
    y._update(ys)
    return y


@dataclass
class RoundInfo:
    ranks: tuple
    sigma1: np.ndarray
    sigma2: np.ndarray
    discarded: tuple
    norm: float


def tt_round(x: TT, tol: float, rmax: int = 0, ctx: Context | None = None,
             want_info: bool = False):
    """In-place TT rounding T_tol (tk_round).  Returns x (and a RoundInfo)."""
    ctx = ctx or default_context()
    s = x.struct()
    D = ctypes.c_double
    if ctx.async_on:
        if want_info:
            raise ValueError("want_info needs a synchronous context")
        ctx.check(lib().tk_round(ctx._h, ctypes.byref(s), float(tol), int(rmax), None, None, None,
                                 None))
        x._queue(ctx, s)
        return x
    if want_info:
        s1 = (D * max(x.r1, 1))()
        s2 = (D * max(x.r2, 1))()
        disc = (D * 2)()
        nrm = D()
        ctx.check(lib().tk_round(ctx._h, ctypes.byref(s), float(tol), int(rmax), s1, s2, disc,
                                 ctypes.byref(nrm)))
    else:
        ctx.check(lib().tk_round(ctx._h, ctypes.byref(s), float(tol), int(rmax), None, None, None,
                                 None))
    x._update(s)
    if want_info:
        return x, RoundInfo((x.r1, x.r2), np.array(s1[:]), np.array(s2[:]), (disc[0], disc[1]),
                            nrm.value)
    return x


def tt_apply_round(op: "Operator", x: TT, tol: float, rmax: int = 0, out: TT | None = None,
                   want_info: bool = False):
    """y = T_tol(A x) fused (tk_apply_round): the block-diagonal middle core of A x is never
    written densely.  Same results as tt_round(tt_apply_op(op, x), tol, rmax)."""
    ctx = op.ctx
    T = op.T
    y = out if out is not None else TT(x.n_x, x.n_xi, x.n_t, T * x.r1, T * x.r2)
    xs, ys = x.struct(), y.struct()
    D = ctypes.c_double
    if ctx.async_on:
        if want_info:
            raise ValueError("want_info needs a synchronous context")
        ctx.check(lib().tk_apply_round(ctx._h, op._h, ctypes.byref(xs), ctypes.byref(ys),
                                       float(tol), int(rmax), None, None, None, None))
        y._queue(ctx, ys)
        ctx._pending.append((None, xs))  # keeps the input struct alive until sync
        return y
    if want_info:
        s1 = (D * max(T * x.r1, 1))()
        s2 = (D * max(T * x.r2, 1))()
        disc = (D * 2)()
        nrm = D()
        ctx.check(lib().tk_apply_round(ctx._h, op._h, ctypes.byref(xs), ctypes.byref(ys),
                                       float(tol), int(rmax), s1, s2, disc, ctypes.byref(nrm)))
    else:
        ctx.check(lib().tk_apply_round(ctx._h, op._h, ctypes.byref(xs), ctypes.byref(ys),
                                       float(tol), int(rmax), None, None, None, None))
    y._update(ys)
    if want_info:
        return y, RoundInfo((y.r1, y.r2), np.array(s1[:]), np.array(s2[:]), (disc[0], disc[1]),
                            nrm.value)
    return y


def tt_dot(x: TT, y: TT, ctx: Context | None = None, out: torch.Tensor | None = None):
    """<x, y>_F into a 1-element device tensor (tk_dot); .item() syncs."""
    ctx = ctx or default_context()
    out = out if out is not None else torch.empty(1, dtype=torch.float64, device="cuda")
    xs, ys = x.struct(), y.struct()
    ctx.check(lib().tk_dot(ctx._h, ctypes.byref(xs), ctypes.byref(ys), ctypes.c_void_p(out.data_ptr())))
    return out


def tt_norm(x: TT, ctx: Context | None = None, out: torch.Tensor | None = None):
    ctx = ctx or default_context()
    out = out if out is not None else torch.empty(1, dtype=torch.float64, device="cuda")
    xs = x.struct()
    ctx.check(lib().tk_norm(ctx._h, ctypes.byref(xs), ctypes.c_void_p(out.data_ptr())))
    return out


def tt_axpby(a, x: TT, b, y: TT, ctx: Context | None = None, out: TT | None = None) -> TT:
    """z = a x + b y (tk_axpby / tk_axpby_host); a, b floats or 1-element device tensors."""
    ctx = ctx or default_context()
    z = out or TT(x.n_x, x.n_xi, x.n_t, x.r1 + y.r1, x.r2 + y.r2)
    xs, ys, zs = x.struct(), y.struct(), z.struct()
    if isinstance(a, torch.Tensor) or isinstance(b, torch.Tensor):
        at = a if isinstance(a, torch.Tensor) else torch.tensor([float(a)], dtype=torch.float64, device="cuda")
        bt = b if isinstance(b, torch.Tensor) else torch.tensor([float(b)], dtype=torch.float64, device="cuda")
        ctx.check(lib().tk_axpby(ctx._h, ctypes.c_void_p(at.data_ptr()), ctypes.byref(xs),
                                 ctypes.c_void_p(bt.data_ptr()), ctypes.byref(ys), ctypes.byref(zs)))
    else:
        ctx.check(lib().tk_axpby_host(ctx._h, float(a), ctypes.byref(xs), float(b), ctypes.byref(ys),
                                      ctypes.byref(zs)))
    z._update(zs)
    return z


def gmres_cycle(op: Operator, b: TT, steps: int = 20, tol: float = 1e-6, prec=None):
    """One low-rank GMRES cycle (tk_gmres_cycle; tk_gmres_cycle_p with a MeanLSC prec: flexible
    right preconditioning).  Returns dict(history, steps, explicit, step_ms)."""
    ctx = op.ctx
    D = ctypes.c_double
    hist = (D * (steps + 1))()
    ms = (D * steps)()
    done = ctypes.c_int()
    expl = D()
    bs = b.struct()
    if prec is None:
        ctx.check(lib().tk_gmres_cycle(ctx._h, op._h, ctypes.byref(bs), int(steps), float(tol),
                                       hist, ctypes.byref(done), ctypes.byref(expl), ms))
    else:
        ctx.check(lib().tk_gmres_cycle_p(ctx._h, op._h, prec._h, ctypes.byref(bs), int(steps),
                                         float(tol), hist, ctypes.byref(done), ctypes.byref(expl),
                                         ms))
    k = done.value
    return dict(history=np.array(hist[: k + 1]), steps=k, explicit=expl.value,
                step_ms=np.array(ms[:k]))


def gmres_solve(op: Operator, b: TT, restart: int = 20, max_cycles: int = 5, tol: float = 1e-6,
                tol_gmres: float = 1e-8, eps_soln: float = -1.0, cap: tuple | None = None,
                prec=None):
    """Complete restarted low-rank GMRES (tk_gmres_solve; Alg. 3 + eq:eps_soln, P = I).
    Returns dict(z, explicit, ls, cycles, steps).  cap: rank capacity of z (default bounded by
    the mode sizes and 512)."""
    ctx = op.ctx
    if cap is None:
        cap = (max(1, min(b.n_x, b.n_xi * b.n_t, 512)), max(1, min(b.n_t, b.n_x * b.n_xi, 512)))
    z = TT(b.n_x, b.n_xi, b.n_t, cap[0], cap[1])
    D = ctypes.c_double
    expl = (D * (max_cycles + 1))()
    ls = (D * (max(max_cycles, 1) * (restart + 1)))()
    steps = (ctypes.c_int * max(max_cycles, 1))()
    done = ctypes.c_int()
    bs, zs = b.struct(), z.struct()
    args = (ctypes.byref(bs), int(restart), int(max_cycles), float(tol), float(tol_gmres),
            float(eps_soln), ctypes.byref(zs), expl, ls, ctypes.byref(done), steps)
    if prec is None:
        ctx.check(lib().tk_gmres_solve(ctx._h, op._h, *args))
    else:
        ctx.check(lib().tk_gmres_solve_p(ctx._h, op._h, prec._h, *args))
    z._update(zs)
    c = done.value
    lsv = np.array(ls[: c * (restart + 1)]).reshape(c, restart + 1) if c else np.zeros((0, restart + 1))
    return dict(z=z, explicit=np.array(expl[: c + 1]), cycles=c, steps=list(steps[:c]),
                ls=[row[: steps[i] + 1] for i, row in enumerate(lsv)])


# ----------------------------------------------------------------------------- NEXT-3
def _csr_arrays(m):
    rp = np.ascontiguousarray(m.indptr, dtype=np.int32)
    cl = np.ascontiguousarray(m.indices, dtype=np.int32)
    vl = np.ascontiguousarray(m.data, dtype=np.float64)
    return rp, cl, vl


def _default_cap(n_x, n_xi, n_t):
    return (max(1, min(n_x, n_xi * n_t, 1024)), max(1, min(n_t, n_x * n_xi, 1024)))


class BlockTridiag:
    """Block-tridiagonal direct solver of a spatial factor (tk_bt_create / _gram): K = A + shift I
    (gram=False) or K = A A^T (gram=True) for the scipy CSR A, blocks of N rows."""

    def __init__(self, A, nb: int, N: int, shift: float = 0.0, gram: bool = False,
                 ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.n = int(nb) * int(N)
        rp, cl, vl = _csr_arrays(A)
        self._h = ctypes.c_void_p()
        if gram:
            rc = lib().tk_bt_create_gram(self.ctx._h, ctypes.byref(self._h), int(nb), int(N),
                                         int(A.shape[1]), rp.ctypes.data, cl.ctypes.data,
                                         vl.ctypes.data)
        else:
            rc = lib().tk_bt_create(self.ctx._h, ctypes.byref(self._h), int(nb), int(N),
                                    rp.ctypes.data, cl.ctypes.data, vl.ctypes.data, float(shift))
        self.ctx.check(rc)

    def solve(self, x: TT, row0: int = 0, reps: int = 1) -> TT:
        """(I (x) I (x) K^{-1}) x on rows [row0, row0 + reps n) of the space core, zero elsewhere."""
        y = TT(x.n_x, x.n_xi, x.n_t, x.r1, x.r2)
        xs, ys = x.struct(), y.struct()
        self.ctx.check(lib().tk_bt_solve(self.ctx._h, self._h, ctypes.byref(xs), int(row0),
                                         int(reps), ctypes.byref(ys)))
        y._update(ys)
        return y

    def __del__(self):
        try:
            if self._h:
                lib().tk_bt_destroy(self._h)
        except Exception:
            pass


class MeanLSC:
    """P^{-1} of eq:prec with S_LSC,0 (eq:mean_lsc) and the inner (F0 + C) GMRES preconditioned
    by M (eq:11_prec), tk_prec_create_lsc.  F0s (n_v x n_v) and B (n_p x 2 n_v) scipy CSR."""

    def __init__(self, F0s, B, tau: float, n_xi: int, n_t: int, tol: float, grid: int,
                 tol_in: float = 1e-1, restart_in: int = 10, max_cycles_in: int = 3,
                 ctx: Context | None = None):
        self.ctx = ctx or default_context()
        self.n_x = 2 * F0s.shape[0] + B.shape[0]
        self.n_xi, self.n_t = int(n_xi), int(n_t)
        f = _csr_arrays(F0s)
        b = _csr_arrays(B)
        self._h = ctypes.c_void_p()
        self.ctx.check(lib().tk_prec_create_lsc(
            self.ctx._h, ctypes.byref(self._h), self.n_xi, self.n_t, int(grid),
            f[0].ctypes.data, f[1].ctypes.data, f[2].ctypes.data,
            b[0].ctypes.data, b[1].ctypes.data, b[2].ctypes.data,
            float(tau), float(tol), float(tol_in), int(restart_in), int(max_cycles_in)))

    def apply(self, v: TT, part: int = 0, cap: tuple | None = None) -> TT:
        """part 0: P^{-1} v; 1: M^{-1} v (eq:11_prec); 2: S_LSC,0^{-1} v_p (eq:mean_lsc)."""
        cap = cap or _default_cap(v.n_x, v.n_xi, v.n_t)
        out = TT(v.n_x, v.n_xi, v.n_t, 1, 1, cap[0], cap[1])
        vs, os_ = v.struct(), out.struct()
        self.ctx.check(lib().tk_prec_apply(self.ctx._h, self._h, int(part), ctypes.byref(vs),
                                           ctypes.byref(os_)))
        out._update(os_)
        return out

    def operator(self, which: int) -> Operator:
        """A borrowed view of the preconditioner's operators: 0 = F0 + C, 1 = B^T, 2 = B."""
        h = lib().tk_prec_operator(self._h, int(which))
        if not h:
            raise TkError(TK_EARG, "tk_prec_operator")
        return _Borrowed(self, h)

    def __del__(self):
        try:
            if self._h:
                lib().tk_prec_destroy(self._h)
        except Exception:
            pass


class _Borrowed(Operator):
    """An operator handle owned by another object (never destroyed here)."""

    def __init__(self, owner, h):
        self.owner = owner  # keeps the owner (and so the handle) alive
        self.ctx, self.n_x, self.n_xi, self.n_t = owner.ctx, owner.n_x, owner.n_xi, owner.n_t
        self._h = ctypes.c_void_p(h)
        self.T = int(lib().tk_op_terms(self._h))

    def __del__(self):
        pass


# ----------------------------------------------------------------------------- NEXT-4
def picard(stokes: Operator, conv: Convection, f: TT, tol_picard: float = 1e-4, maxit: int = 10,
           tol_gmres: float = 1e-1, eps_gmres: float = 1e-3, eps_conv: float = -1.0,
           restart: int = 20, max_cycles: int = 5, prec: "MeanLSC | None" = None,
           cap: tuple | None = None):
    """Inexact Picard iteration of Alg. 1 (tk_picard).  Returns dict(z, residuals, iterations,
    ranks)."""
    ctx = stokes.ctx
    cap = cap or _default_cap(f.n_x, f.n_xi, f.n_t)
    z = TT(f.n_x, f.n_xi, f.n_t, 1, 1, cap[0], cap[1])
    res = (ctypes.c_double * (maxit + 1))()
    rk = (ctypes.c_int64 * (2 * (maxit + 1)))()
    it = ctypes.c_int()
    fs, zs = f.struct(), z.struct()
    ctx.check(lib().tk_picard(ctx._h, stokes._h, conv._h, prec._h if prec is not None else None,
                              ctypes.byref(fs), float(tol_picard), int(maxit), float(tol_gmres),
                              float(eps_gmres), float(eps_conv), int(restart), int(max_cycles),
                              ctypes.byref(zs), res, ctypes.byref(it), rk))
    z._update(zs)
    n = it.value
    return dict(z=z, residuals=np.array(res[: n + 1]), iterations=n,
                ranks=[(rk[2 * i], rk[2 * i + 1]) for i in range(n + 1)])


def round_workspace_bytes(n_x, n_xi, n_t, R1, R2) -> int:
    """tk_round_workspace_bytes: scratch bound of one rounding on grown ranks (R1, R2)."""
    return int(lib().tk_round_workspace_bytes(int(n_x), int(n_xi), int(n_t), int(R1), int(R2)))
