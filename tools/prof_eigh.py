"""Time the eigh comparison route vs solve_chol at a given shape (device-resident fp32 scores)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2310_17556_b200 as fsb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
dev = torch.device("cuda", 0)
S = torch.randn(n, m, device=dev) / n ** 0.5
v = torch.randn(m, device=dev)
system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
for prec in ("f16x2", "fp64"):
    for route in ("chol", "eigh", "svd"):
        f = {"chol": fsb.solve_chol, "eigh": fsb.solve_svd_eigh, "svd": fsb.solve_svd_direct}[route]
        f(system, precision=prec)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sol = f(system, precision=prec)
        torch.cuda.synchronize()
        print(f"{route:5s} {prec:6s} n={n} m={m}: {1e3 * (time.perf_counter() - t0):8.2f} ms  rel_res {sol.rel_residual:.2e}")
w, U, sweeps = fsb.eigh_gram(fsb.ScoreMatrix(S[:, :100000]), "fp64")
torch.cuda.synchronize()
t0 = time.perf_counter()
w, U, sweeps = fsb.eigh_gram(fsb.ScoreMatrix(S[:, :100000]), "fp64")
torch.cuda.synchronize()
print(f"eigh_gram n={n} (m=1e5 Gram + Jacobi): {1e3 * (time.perf_counter() - t0):.2f} ms, {sweeps} sweeps")
