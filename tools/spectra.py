"""Print the bond spectra tk_round sees at a config (diagnostic)."""
import sys

import numpy as np
import torch

import paper_1906_06785_b200 as ttk
from synth.configs import CONFIGS
from synth.operator import build_operator
from synth.tt import make_input_tt

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
op = build_operator(cfg)
x = make_input_tt(cfg, op.n_xi)
gop = ttk.Operator.from_kronsum(op)
y = ttk.tt_apply_op(gop, ttk.TT.from_cores(*x))
g, info = ttk.tt_round(y, cfg.tol, cfg.rmax, want_info=True)
print("ranks", g.ranks, "norm", info.norm, "disc", info.discarded)
for name, s in (("sigma1", info.sigma1), ("sigma2", info.sigma2)):
    s = np.asarray(s)
    s = s[s > 0]
    rel = s / s[0]
    dec = [int(np.sum(rel > 10.0 ** (-d))) for d in range(0, 17, 2)]
    print(name, len(s), "count above 1e-0,-2,...,-16:", dec)
