"""Print the library's per-kernel timeline of ONE c4 apply+round (tk_ctx_profile(ctx, 3) profiling dump):
start offset, duration and phase of every profiled launch, to see what overlaps and where the
GPU idles on the latency-bound chain.  usage: python tools/timeline.py [config] > out.txt"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1906_06785_b200 as ttk  # noqa: E402
from paper_1906_06785_b200 import ttk as ttkmod  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from synth.operator import build_operator  # noqa: E402
from synth.tt import make_input_tt  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
op = build_operator(cfg)
x = make_input_tt(cfg, op.n_xi)
ctx = ttk.default_context()
gop = ttk.Operator.from_kronsum(op, ctx)
xg = ttk.TT.from_cores(*x)
ycap = ttk.TT(op.n_x, op.n_xi, op.n_t, op.T * xg.r1, op.T * xg.r2)
L = ttkmod.lib()
for i in range(3):
    if i == 2:
        L.tk_ctx_profile(ctx._h, 3)
    ttk.tt_apply_round(gop, xg, cfg.tol, cfg.rmax, out=ycap)
    torch.cuda.synchronize()
buf = ctypes.create_string_buffer(1 << 24)
L.tk_ctx_profile_dump(ctx._h, buf, len(buf))
rows = [ln.split() for ln in buf.value.decode().splitlines()]
rows.sort(key=lambda r: float(r[4]))
end = 0.0
for cat, ms, fl, by, t0 in rows:
    t0, ms = float(t0), float(ms)
    gap = t0 - end
    print(f"{t0:9.3f} {ms:8.3f} {'gap %.3f' % gap if gap > 0.02 else '':>10s} {cat}")
    end = max(end, t0 + ms)
print(f"total {end:.3f} ms")
