"""Why is the pipelined c4 e2e step slower than the device step?  Per-op times of back-to-back
tk_apply_round calls: alone, alternating output buffers, with concurrent H2D / D2H copies."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1906_06785_b200 as ttk
from synth.configs import CONFIGS
from synth.operator import build_operator
from synth.tt import make_input_tt
cfg = CONFIGS["c4"]; op = build_operator(cfg); x = make_input_tt(cfg, op.n_xi)
ctx = ttk.default_context(); gop = ttk.Operator.from_kronsum(op, ctx); T = op.T
xs = [ttk.TT.from_cores(*x) for _ in range(2)]
ys = [ttk.TT(op.n_x, op.n_xi, op.n_t, T * 64, T * 64) for _ in range(2)]
st = torch.cuda.current_stream()
def run(label, nbuf, h2d=False, d2h=False, n=5):
    pinned = [torch.from_numpy(np.ascontiguousarray(c)).pin_memory() for c in x]
    outs = torch.empty(op.n_x * 160, dtype=torch.float64).pin_memory()
    s2 = torch.cuda.Stream()
    for _ in range(2):
        ttk.tt_apply_round(gop, xs[0], cfg.tol, cfg.rmax, out=ys[0])
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    t0 = time.perf_counter()
    for i in range(n):
        if h2d:
            with torch.cuda.stream(s2):
                xs[(i + 1) % nbuf].b1[: pinned[0].numel()].copy_(pinned[0].reshape(-1), non_blocking=True)
        ev[i][0].record(st)
        y = ttk.tt_apply_round(gop, xs[i % nbuf], cfg.tol, cfg.rmax, out=ys[i % nbuf])
        ev[i][1].record(st)
        if d2h:
            done = torch.cuda.Event(); done.record(st)
            with torch.cuda.stream(s2):
                s2.wait_event(done)
                outs.copy_(ys[i % nbuf].b1[: outs.numel()], non_blocking=True)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / n
    print(f"{label:34s} per-op events {[round(a.elapsed_time(b), 1) for a, b in ev]}  wall/op {wall:.1f} ms", flush=True)
run("1 buffer, no copies", 1)
run("2 buffers, no copies", 2)
run("2 buffers, H2D of next input", 2, h2d=True)
run("2 buffers, D2H of result", 2, d2h=True)
run("2 buffers, H2D + D2H", 2, h2d=True, d2h=True)
