"""Two tk_gemm calls of the same kernel instantiation running concurrently on two streams:
each result must equal its stand-alone result bitwise."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1906_06785_b200 as ttk

g = torch.Generator(device="cuda").manual_seed(1)
M1, N1, K1 = 196608, 120, 320
M2, N2, K2 = 30240, 80, 360
A1 = torch.randn((M1, K1), dtype=torch.float64, device="cuda", generator=g)
B1 = torch.randn((K1, N1), dtype=torch.float64, device="cuda", generator=g)
A2 = torch.randn((M2, K2), dtype=torch.float64, device="cuda", generator=g)
B2 = torch.randn((K2, N2), dtype=torch.float64, device="cuda", generator=g)
for feed in (1, 0):
    s1 = torch.cuda.Stream(priority=0)
    s2 = torch.cuda.Stream(priority=-1)
    c1 = ttk.Context(s1); c1.set_gemm_feed(feed)
    c2 = ttk.Context(s2); c2.set_gemm_feed(feed)
    R1 = torch.empty((M1, N1), dtype=torch.float64, device="cuda")
    R2 = torch.empty((M2, N2), dtype=torch.float64, device="cuda")
    c1.gemm(A1, B1, R1, M1, N1, K1); torch.cuda.synchronize()
    c2.gemm(A2, B2, R2, M2, N2, K2); torch.cuda.synchronize()
    bad1 = bad2 = 0
    for rep in range(10):
        C1 = torch.full((M1, N1), float("nan"), dtype=torch.float64, device="cuda")
        C2s = [torch.full((M2, N2), float("nan"), dtype=torch.float64, device="cuda") for _ in range(6)]
        torch.cuda.synchronize()
        c1.gemm(A1, B1, C1, M1, N1, K1)
        for C2 in C2s:
            c2.gemm(A2, B2, C2, M2, N2, K2)
        torch.cuda.synchronize()
        bad1 += int(not torch.equal(C1, R1))
        bad2 += sum(int(not torch.equal(C2, R2)) for C2 in C2s)
        if not torch.equal(C1, R1):
            d = (C1 - R1).abs(); idx = d.nonzero()
            print("   C1 diff n", idx.shape[0], "rows", idx[:, 0].min().item(), idx[:, 0].max().item(), "cols", sorted(set(idx[:, 1].tolist()))[:20], "max", d.max().item())
    print(f"feed={feed}: concurrent mismatches big={bad1}/10 small={bad2}/60", flush=True)
