"""fp64-mode Gram accuracy against exactly rounded sums (math.fsum of exact fp64 products of fp32
scores) for a sample of entries, next to numpy's dgemm; and the fp64 solve's first-pass residual
(refine=False) vs the automatic rule. n m (default 1024 1e6)."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2310_17556_b200 as fsb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
rng = np.random.Generator(np.random.PCG64(0))
S = rng.standard_normal((n, m), dtype=np.float32) / np.float32(np.sqrt(n))
v = rng.standard_normal(m).astype(np.float32)
A = S.astype(np.float64)
St = torch.from_numpy(S).cuda()
Wg = fsb.gram(fsb.ScoreMatrix(St), 1e-300, precision="fp64")
Wg = Wg.cpu().numpy() if hasattr(Wg, "cpu") else np.asarray(Wg)
pairs = [(i, i) for i in range(0, n, max(1, n // 11))] + [(i, (i * 7 + 3) % n) for i in range(0, n, max(1, n // 12))]
eo, en = [], []
for i, j in pairs:
    ex = math.fsum((A[i] * A[j]).tolist())
    eo.append(abs(Wg[i, j] - ex) / abs(Wg[i, i]))
    en.append(abs(float(A[i] @ A[j]) - ex) / abs(Wg[i, i]))
print(f"n={n} m={m} gram error / diag: ours max {max(eo):.2e} mean {np.mean(eo):.2e} | "
      f"numpy dot max {max(en):.2e} mean {np.mean(en):.2e}", flush=True)
system = fsb.DampedSystem(fsb.ScoreMatrix(St), 1e-3, torch.from_numpy(v).cuda())
a = fsb.solve_chol(system, precision="fp64", refine=False)
b = fsb.solve_chol(system, precision="fp64")
print(f"fp64 solve rel_residual: first pass {a.rel_residual:.2e}, auto rule {b.rel_residual:.2e}", flush=True)
