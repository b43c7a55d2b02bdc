"""Time tk_gemm on the c4 heavy shapes with both operand feeds (TMA tensor tiles vs cp.async).
Diagnostic: python tools/ubench/gemm_feed.py [reps]  ->  one line per (shape, feed)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1906_06785_b200 as ttk  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n_x = 786432
SHAPES = [  # name, M, N, K, transA, transB, sym
    ("form_W  (n_x x 640 x 896)", n_x, 640, 896, False, False, False),
    ("gram_W  (sym 640 x 640 x n_x)", 640, 640, n_x, True, False, True),
    ("form_U1 (n_x x 160 x 640)", n_x, 160, 640, False, False, False),
    ("gram_Y  (sym 896 x 896 x n_x/16)", 896, 896, n_x // 16, True, False, True),
    ("dot W1  (448 x 320 x n_x)", 448, 320, n_x, True, False, False),
]
g = torch.Generator(device="cuda").manual_seed(1)
for name, M, N, K, ta, tb, sym in SHAPES:
    A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda", generator=g)
    B = A if sym else torch.randn((N, K) if tb else (K, N), dtype=torch.float64, device="cuda", generator=g)
    C = torch.empty((M, N), dtype=torch.float64, device="cuda")
    flops = (M * (M + 1) * K) if sym else 2.0 * M * N * K
    res = {}
    for feed in (0, 1):
        ctx = ttk.Context()
        ctx.set_gemm_feed(feed)
        ctx.gemm(A, B, C, M, N, K, trans_a=ta, trans_b=tb, sym=sym)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            ctx.gemm(A, B, C, M, N, K, trans_a=ta, trans_b=tb, sym=sym)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        res[feed] = C.clone()
        print(f"{name:34s} feed={'tma' if feed else 'cp.async':8s} {ms:8.3f} ms  {flops / ms / 1e9:6.2f} TF/s (algorithmic)", flush=True)
    d = (res[0] - res[1]).abs().max().item()
    print(f"   max |cp.async - tma| = {d:.3e} (max |C| {res[0].abs().max().item():.3e})", flush=True)
    del A, B, C, res
