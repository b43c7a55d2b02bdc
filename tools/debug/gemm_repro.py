"""Bitwise run-to-run reproducibility of tk_gemm (both feeds) on rounding-like shapes."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1906_06785_b200 as ttk

g = torch.Generator(device="cuda").manual_seed(1)
SH = [("gramY sampled", 360, 360, 196608 // 16, True, False, True, 16 * 360),
      ("formW", 196608, 280, 360, False, False, False, None),
      ("gramW", 280, 280, 196608, True, False, True, None),
      ("formU1", 196608, 120, 280, False, False, False, None),
      ("mid", 360, 21504, 360, False, False, False, None),
      ("gramC", 128, 128, 10080, True, False, True, None),
      ("wide", 360, 360, 21504, False, True, True, None)]
for feed in (1, 0):
    ctx = ttk.Context(); ctx.set_gemm_feed(feed)
    for name, M, N, K, ta, tb, sym, lda in SH:
        A = torch.randn(((K, lda or M) if ta else (M, lda or K)), dtype=torch.float64, device="cuda", generator=g)
        B = A if sym else torch.randn((N, K) if tb else (K, N), dtype=torch.float64, device="cuda", generator=g)
        outs = []
        for rep in range(6):
            C = torch.full((M, N), float("nan"), dtype=torch.float64, device="cuda")
            ctx.gemm(A, B, C, M, N, K, trans_a=ta, trans_b=tb, sym=sym, lda=lda, ldb=(lda if sym else None))
            torch.cuda.synchronize()
            outs.append(C)
        bad = [i for i in range(1, 6) if not torch.equal(outs[0], outs[i])]
        nan = bool(torch.isnan(outs[0]).any())
        print(f"feed={feed} {name:14s} mismatching reps {bad} nan={nan}", flush=True)
        if bad:
            d = (outs[0] - outs[bad[0]]).abs()
            idx = d.nonzero()
            print("   n diff", idx.shape[0], "first", idx[:5].tolist(), "max", d.max().item())
