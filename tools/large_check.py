import sys, time; sys.path.insert(0, "/root/repo")
import torch, numpy as np
import paper_2310_17556_b200 as fsb
dev = torch.device("cuda", 0)
for n, m in ((2048, 500000), (4096, 300000), (3000, 123457)):
    g = torch.Generator(device=dev).manual_seed(n)
    S = torch.randn(n, m, device=dev, generator=g) / n ** 0.5
    v = torch.randn(m, device=dev, generator=g)
    system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
    out = {}
    for prec in ("f16x2", "tf32x3", "fp64"):
        fsb.solve_chol(system, precision=prec)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        sol = fsb.solve_chol(system, precision=prec)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        out[prec] = sol
        print(f"n={n} m={m} {prec:6s} {1e3*dt:8.2f} ms rel_res {sol.rel_residual:.2e}", flush=True)
    for prec in ("f16x2", "tf32x3"):
        d = (out[prec].x - out["fp64"].x).norm() / out["fp64"].x.norm()
        print(f"   {prec} vs fp64 relerr {d.item():.2e}")
    del S, v, system, out
    torch.cuda.empty_cache()
