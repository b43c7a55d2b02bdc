"""Per-phase device time and host-side gaps of one c5 low-rank GMRES cycle (tk_ctx_profile(ctx, 3)):
where a Krylov step's time goes.  usage: python tools/gmres_profile.py"""
import collections
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1906_06785_b200 as ttk  # noqa: E402
from paper_1906_06785_b200 import ttk as ttkmod  # noqa: E402
from synth.configs import CONFIGS  # noqa: E402
from synth.operator import build_operator  # noqa: E402
from synth.tt import make_rhs_tt  # noqa: E402

cfg = CONFIGS["c5"]
op = build_operator(cfg)
b = make_rhs_tt(cfg, op.n_xi)
ctx = ttk.default_context()
gop = ttk.Operator.from_kronsum(op, ctx)
bg = ttk.TT.from_cores(*b)
ttk.gmres_cycle(gop, bg, 4, cfg.tol)
torch.cuda.synchronize()
L = ttkmod.lib()
L.tk_ctx_profile(ctx._h, 3)
t0 = time.perf_counter()
res = ttk.gmres_cycle(gop, bg, cfg.gmres_steps, cfg.tol)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
buf = ctypes.create_string_buffer(1 << 26)
n = L.tk_ctx_profile_dump(ctx._h, buf, len(buf))
rows = [ln.split() for ln in buf.value.decode().splitlines()]
agg = collections.defaultdict(lambda: [0, 0.0])
end = 0.0
busy = 0.0
for cat, ms, fl, by, t in sorted(rows, key=lambda r: float(r[4])):
    agg[cat][0] += 1
    agg[cat][1] += float(ms)
    s0, ms = float(t), float(ms)
    busy += max(0.0, min(s0 + ms, max(end, s0 + ms)) - max(s0, end))
    end = max(end, s0 + ms)
print(f"wall {wall * 1e3:.1f} ms, device span {end:.1f} ms, busy (union of records) {busy:.1f} ms,"
      f" records {n}, launches {ctx.launches}")
for cat, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {cat:18s} n={c:6d} {ms:10.2f} ms")
print("steps ms:", [round(v, 1) for v in res["step_ms"]])
