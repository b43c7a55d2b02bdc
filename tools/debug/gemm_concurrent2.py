"""tk_gemm (TMA feed) on a low-priority stream while another context rounds a c2 TT (Jacobi,
panels, small GEMMs) on a high-priority stream: result vs stand-alone result; per-k-tile
attribution of any difference."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1906_06785_b200 as ttk
from synth.configs import CONFIGS
from synth.operator import build_operator
from synth.tt import make_input_tt

cfg = CONFIGS["c2"]
op = build_operator(cfg)
x = make_input_tt(cfg, op.n_xi)
g = torch.Generator(device="cuda").manual_seed(1)
M, N, K = 196608, 120, 320
A = torch.randn((M, K), dtype=torch.float64, device="cuda", generator=g)
B = torch.randn((K, N), dtype=torch.float64, device="cuda", generator=g)
s_lo = torch.cuda.Stream(priority=0)
s_hi = torch.cuda.Stream(priority=-1)
c_lo = ttk.Context(s_lo)
with torch.cuda.stream(s_hi):
    c_hi = ttk.Context(s_hi)
    gop = ttk.Operator.from_kronsum(op, c_hi)
    xg = ttk.TT.from_cores(*x)
    y0 = ttk.tt_apply_op(gop, xg)
    base = [torch.as_tensor(c).clone() for c in (y0.U1, y0.U2, y0.U3)]
torch.cuda.synchronize()
for feed in (1, 0):
    c_lo.set_gemm_feed(feed)
    R = torch.empty((M, N), dtype=torch.float64, device="cuda")
    c_lo.gemm(A, B, R, M, N, K); torch.cuda.synchronize()
    nbad = 0
    for rep in range(8):
        C = torch.full((M, N), float("nan"), dtype=torch.float64, device="cuda")
        with torch.cuda.stream(s_hi):
            y = ttk.TT.from_cores(*[b.clone() for b in base])
        torch.cuda.synchronize()
        for _ in range(3):
            c_lo.gemm(A, B, C, M, N, K)
        with torch.cuda.stream(s_hi):
            ttk.tt_round(y, cfg.tol, cfg.rmax, ctx=c_hi)
        c_lo.gemm(A, B, C, M, N, K)
        torch.cuda.synchronize()
        if not torch.equal(C, R):
            nbad += 1
            d = (C - R).abs(); idx = d.nonzero()
            r0, c0 = idx[0].tolist()
            print(f"  rep {rep}: ndiff {idx.shape[0]} rows [{idx[:,0].min().item()},{idx[:,0].max().item()}] first ({r0},{c0}) got {C[r0,c0].item():.6g} want {R[r0,c0].item():.6g}")
            # per-k-tile attribution for the first bad element
            a = A[r0].cpu().numpy(); b = B[:, c0].cpu().numpy()
            diff = C[r0, c0].item() - R[r0, c0].item()
            terms = [(t, float(np.dot(a[16*t:16*t+16], b[16*t:16*t+16]))) for t in range(K // 16)]
            print("     diff", diff, "k-tile sums", [f"{v:.3g}" for _, v in terms][:20])
    print(f"feed={feed}: {nbad}/8 concurrent runs differ", flush=True)
