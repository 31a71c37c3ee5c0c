"""Refinement behaviour at the headline shape (n=1024, m=1e6, lam=1e-3, the bench's PCG64 system):
rel_residual and relerr(x) vs the CPU reference after k correction steps, per precision mode, with
device times.  python tools/refine_headline.py [n m lam]"""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import torch
from oracle import fisher_oracle as O
import paper_2310_17556_b200 as fsb

n, m, lam = (int(sys.argv[1]), int(float(sys.argv[2])), float(sys.argv[3])) if len(sys.argv) > 3 else (1024, 1_000_000, 1e-3)
S, v, _ = O.generate_problem(0, n, m, lam)
S32, v32 = S.astype(np.float32), v.astype(np.float32)
np.copyto(S, S32)
ref = O.solve_chol(S, v32.astype(np.float64), lam)
del S
dev = torch.device("cuda", 0)
system = fsb.DampedSystem(fsb.ScoreMatrix(torch.from_numpy(S32).to(dev)), lam, torch.from_numpy(v32).to(dev))
for prec in ("f16x2", "tf32x3", "fp64"):
    out = []
    for k in ((0, 1, 2, 3, 4) if prec != "fp64" else (0, 1)):
        fsb.solve_chol(system, precision=prec, refine=k)
        torch.cuda.synchronize()
        t = time.perf_counter()
        sol = fsb.solve_chol(system, precision=prec, refine=k)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t) * 1e3
        out.append(f"{k}:{sol.rel_residual:.2e}/{O.rel_err(sol.x.cpu().numpy(), ref.x):.1e}/{ms:.1f}ms")
    print(prec, " ".join(out), flush=True)
t = time.perf_counter()
sol = fsb.solve_chol(system)
torch.cuda.synchronize()
print("auto:", sol.precision, f"{sol.rel_residual:.2e}", f"{O.rel_err(sol.x.cpu().numpy(), ref.x):.1e}",
      f"{(time.perf_counter() - t) * 1e3:.1f} ms")
