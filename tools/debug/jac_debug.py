"""Per-call Jacobi timing (TTK_JAC_DEBUG build) on a synchronous c3 / c4 rounding."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1906_06785_b200 as ttk
from synth.configs import CONFIGS
from synth.operator import build_operator
from synth.tt import make_input_tt

name, js = sys.argv[1], int(sys.argv[2])
cfg = CONFIGS[name]
op = build_operator(cfg)
x = make_input_tt(cfg, op.n_xi)
ctx = ttk.Context(); ctx.set_jacobi_schedule(js)
gop = ttk.Operator.from_kronsum(op, ctx)
xg = ttk.TT.from_cores(*x)
for rep in range(2):
    y = ttk.tt_apply_op(gop, xg)
    torch.cuda.synchronize()
    print(f"--- {name} js={js} rep {rep}", file=sys.stderr, flush=True)
    ttk.tt_round(y, cfg.tol, cfg.rmax, ctx=ctx)
    torch.cuda.synchronize()
    del y
