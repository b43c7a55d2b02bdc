"""Debug driver: the steps of tk_picard one C-ABI call at a time (error triage)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1906_06785_b200 as ttk
from synth import gpc
from synth.configs import CONFIGS
from synth.operator import build_operator, convection_stencils, picard_forcing
cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c7"]
op = build_operator(cfg)
H = gpc.h_matrices(cfg.m, cfg.p)
D, nv = convection_stencils(cfg.grid)
f = picard_forcing(cfg, op.n_xi)
ctx = ttk.default_context()
g_op = ttk.Operator.from_kronsum(op, ctx)
conv = ttk.Convection(op.n_x, op.n_xi, op.n_t, D, nv, np.array(H), ctx=ctx)
ft = ttk.TT.from_cores(*f)
s = ttk.gmres_solve(g_op, ft, restart=20, max_cycles=5, tol=cfg.tol, tol_gmres=0.1)
z = s["z"]
print("stokes solve", s["cycles"], s["explicit"], z.ranks, flush=True)
u = ttk.TT.from_cores(*z.cores_numpy())
ttk.tt_round(u, cfg.tol)
print("u ranks", u.ranks, flush=True)
N = conv.operator(u)
print("N terms", N.T, flush=True)
L = ttk.Operator.concat([g_op, N])
print("L terms", L.T, flush=True)
y = ttk.tt_apply_op(L, z)
print("apply", y.ranks, flush=True)
r = ttk.tt_axpby(1.0, ft, -1.0, y)
print("axpby", r.ranks, flush=True)
ttk.tt_round(r, cfg.tol)
print("round", r.ranks, flush=True)
import ctypes
lib = ttk.lib()
y2 = ttk.tt_apply_op(L, r)
print("apply_op L r", y2.ranks, flush=True)
ttk.tt_round(y2, cfg.tol)
print("unfused round", y2.ranks, flush=True)
lib.tk_ctx_profile(ctx._h, 3)
try:
    y3 = ttk.tt_apply_round(L, r, cfg.tol)
    print("fused", y3.ranks, flush=True)
    lib.tk_ctx_profile(ctx._h, 3)
    s2 = ttk.gmres_solve(L, r, restart=20, max_cycles=5, tol=cfg.tol, tol_gmres=0.1)
    print("solve 2", s2["cycles"], s2["explicit"], flush=True)
except Exception as e:
    print("FUSED FAILED", e, flush=True)
buf = ctypes.create_string_buffer(1 << 22)
n = lib.tk_ctx_profile_dump(ctx._h, buf, len(buf))
lines = buf.value.decode().splitlines()
print(n, "records; last 15:")
print("\n".join(lines[-25:]))
