"""c5 GMRES cycle re-driven from Python through the binding: input ranks and wall time of every
rounding (sizes of the latency-bound factorisations)."""
import os, sys, time, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1906_06785_b200 as ttk
from synth.configs import CONFIGS
from synth.operator import build_operator
from synth.tt import make_rhs_tt
cfg = CONFIGS["c5"]; op = build_operator(cfg); b = make_rhs_tt(cfg, op.n_xi)
ctx = ttk.default_context(); gop = ttk.Operator.from_kronsum(op, ctx)
recs = []
def rnd(x, kind):
    torch.cuda.synchronize(); t = time.perf_counter(); r_in = x.ranks
    ttk.tt_round(x, cfg.tol); torch.cuda.synchronize()
    recs.append((kind, r_in, x.ranks, (time.perf_counter() - t) * 1e3)); return x
import ctypes
from paper_1906_06785_b200 import ttk as _m
L = _m.lib()
NSTEP = int(sys.argv[1]) if len(sys.argv) > 1 else 10
def dump(title):
    buf = ctypes.create_string_buffer(1 << 24)
    n = L.tk_ctx_profile_dump(ctx._h, buf, len(buf)); L.tk_ctx_profile(ctx._h, 0)
    rows = [ln.split() for ln in buf.value.decode().splitlines()]
    agg = collections.defaultdict(lambda: [0, 0.0])
    end = 0.0
    for r in rows:
        agg[r[0]][0] += 1; agg[r[0]][1] += float(r[1]); end = max(end, float(r[4]) + float(r[1]))
    print("==", title, "records", n, f"span {end:.2f} ms")
    for c, (k, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:14]:
        print(f"   {c:16s} n={k:5d} {ms:8.2f} ms")
def apr(v):
    last = len([r for r in recs if r[0] == "apply"]) == NSTEP - 1
    torch.cuda.synchronize(); t = time.perf_counter()
    if last: L.tk_ctx_profile(ctx._h, 3)
    y = ttk.tt_apply_round(gop, v, cfg.tol); torch.cuda.synchronize()
    if last: dump(f"apply round R = {(op.T * v.r1, op.T * v.r2)}")
    recs.append(("apply", (op.T * v.r1, op.T * v.r2), y.ranks, (time.perf_counter() - t) * 1e3)); return y
v0 = rnd(ttk.TT.from_cores(*b), "rhs")
beta = ttk.tt_norm(v0).item(); ttk.tt_axpby(1.0 / beta, v0, 0.0, v0)
V = [ttk.tt_round(ttk.tt_axpby(1.0 / beta, v0, 0.0, v0), 0.0)]
for k in range(NSTEP):
    x = apr(V[k])
    for i in range(k + 1):
        h = ttk.tt_dot(x, V[i]).item()
        last = (k == NSTEP - 1 and i == k)
        if last: L.tk_ctx_profile(ctx._h, 3)
        x = rnd(ttk.tt_axpby(1.0, x, -h, V[i]), "mgs")
        if last: dump(f"mgs round {recs[-1][1]}")
    hn = ttk.tt_norm(x).item()
    V.append(ttk.tt_axpby(1.0 / hn, x, 0.0, x)); V[-1] = ttk.tt_round(V[-1], 0.0)
agg = collections.defaultdict(list)
for kind, ri, ro, ms in recs:
    agg[kind].append(ms)
for kind, ri, ro, ms in recs[-12:]:
    print(kind, ri, "->", ro, f"{ms:.2f} ms")
for k, v in agg.items():
    print(k, len(v), f"total {sum(v):.1f} ms, mean {np.mean(v):.2f}")
