"""Debug driver: one tk_picard run on config c7 (for compute-sanitizer / error triage)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_1906_06785_b200 as ttk
from synth import gpc
from synth.configs import CONFIGS
from synth.operator import build_operator, convection_stencils, picard_forcing
name = sys.argv[1] if len(sys.argv) > 1 else "c7"
cfg = CONFIGS[name]
op = build_operator(cfg)
H = gpc.h_matrices(cfg.m, cfg.p)
D, nv = convection_stencils(cfg.grid)
f = picard_forcing(cfg, op.n_xi)
ctx = ttk.default_context()
g_op = ttk.Operator.from_kronsum(op, ctx)
conv = ttk.Convection(op.n_x, op.n_xi, op.n_t, D, nv, np.array(H), ctx=ctx)
ft = ttk.TT.from_cores(*f)
u = conv.operator(ft)
print("conv op terms", u.T, flush=True)
L = ttk.Operator.concat([g_op, u])
print("concat terms", L.T, flush=True)
y = ttk.tt_apply_op(L, ft)
print("apply ok", y.ranks, flush=True)
g = ttk.picard(g_op, conv, ft, tol_picard=1e-3, maxit=8, tol_gmres=1e-1, eps_gmres=cfg.tol)
print(g["iterations"], g["residuals"], g["ranks"])
