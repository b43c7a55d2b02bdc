"""Bitwise run-to-run reproducibility of tk_round at c3 (sync mode), per GEMM feed."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1906_06785_b200 as ttk
from synth.configs import CONFIGS
from synth.operator import build_operator
from synth.tt import make_input_tt

cfg = CONFIGS["c3"]
op = build_operator(cfg)
x = make_input_tt(cfg, op.n_xi)
for feed in (1, 0):
    ctx = ttk.Context(); ctx.set_gemm_feed(feed)
    gop = ttk.Operator.from_kronsum(op, ctx)
    xg = ttk.TT.from_cores(*x)
    y0 = ttk.tt_apply_op(gop, xg)
    base = [torch.as_tensor(c).clone() for c in (y0.U1, y0.U2, y0.U3)]
    outs = []
    for rep in range(5):
        y = ttk.TT.from_cores(*[b.clone() for b in base])
        torch.cuda.synchronize()
        ttk.tt_round(y, cfg.tol, cfg.rmax, ctx=ctx)
        torch.cuda.synchronize()
        outs.append((y.ranks, [c.copy() for c in y.cores_numpy()]))
    for i in range(1, 5):
        same = outs[i][0] == outs[0][0] and all(np.array_equal(a, b) for a, b in zip(outs[i][1], outs[0][1]))
        md = max(np.abs(a - b).max() for a, b in zip(outs[i][1], outs[0][1])) if outs[i][0] == outs[0][0] else -1
        per = [bool(np.array_equal(a, b)) for a, b in zip(outs[i][1], outs[0][1])]
        print(f"feed={feed} rep {i}: ranks {outs[i][0]} bitwise={same} per-core={per} maxdiff={md:.3e}", flush=True)
