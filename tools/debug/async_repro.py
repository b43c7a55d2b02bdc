"""Async-mode deadlock triage: which host-side action after a queued rounding hangs."""
import faulthandler, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
faulthandler.dump_traceback_later(40, exit=True)
import numpy as np, torch
import paper_1906_06785_b200 as ttk
from synth.configs import CONFIGS
from synth.operator import build_operator
from synth.tt import make_input_tt
mode = sys.argv[1]
cfg = CONFIGS["c2"]
op = build_operator(cfg)
x = make_input_tt(cfg, op.n_xi)
ctx = ttk.Context()
gop = ttk.Operator.from_kronsum(op, ctx)
xg = ttk.TT.from_cores(*x)
y = ttk.tt_apply_op(gop, xg)
torch.cuda.synchronize()
print("on", ctx.set_async(True), flush=True)
ttk.tt_round(y, 1e-10, ctx=ctx)
print("queued 1", flush=True)
if mode == "round2":
    ttk.tt_round(y, 1e-6, ctx=ctx); print("queued 2", flush=True)
if mode == "h2d":
    t = torch.tensor(np.ones(1000), device="cuda"); print("h2d done", flush=True)
if mode == "h2dbig":
    t = ttk.TT.from_cores(*x); print("from_cores done", flush=True)
if mode == "applyround":
    w = ttk.tt_apply_round(gop, xg, cfg.tol, cfg.rmax); print("queued ar", flush=True)
ctx.sync()
print("synced", y.ranks, flush=True)
