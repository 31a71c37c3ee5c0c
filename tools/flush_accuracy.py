"""F16X2 Gram accuracy vs the exact-product fp64 Gram, and the raw / refined solve, at the
headline shape (the kFlushChunks trade-off: fp32 register sums flushed into fp64 every F drains)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2310_17556_b200 as fsb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
g = torch.Generator(device="cuda").manual_seed(5)
S = torch.randn(n, m, device="cuda", generator=g) / n ** 0.5
v = torch.randn(m, device="cuda", generator=g)
sm = fsb.ScoreMatrix(S)
G64 = fsb.gram_packed(sm, 0.0, "fp64")
G16 = fsb.gram_packed(sm, 0.0, "f16x2")
idx = torch.arange(n, device="cuda")
diag = idx * (idx + 1) // 2 + idx
d = (G16 - G64)
rel_diag = (d[diag].abs() / G64[diag].abs()).max().item()
off = d.abs().max().item() / G64[diag].abs().max().item()
system = fsb.DampedSystem(sm, 1e-3, v)
x64 = fsb.solve_chol(system, precision="fp64").x
raw = fsb.solve_chol(system, precision="f16x2", refine=0)
r1 = fsb.solve_chol(system, precision="f16x2", refine=1)
r2 = fsb.solve_chol(system, precision="f16x2", refine=2)
rel = lambda a: ((a - x64).norm() / x64.norm()).item()
print(f"gram max rel diag err {rel_diag:.3e}, max err / max diag {off:.3e}; raw relerr {rel(raw.x):.3e} "
      f"rel_res {raw.rel_residual:.3e}; 1 step {r1.rel_residual:.3e}; 2 steps {r2.rel_residual:.3e}")
