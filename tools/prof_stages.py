"""Per-stage device ms of one solve_chol (fs_profile_enable markers): n m precision [dtype]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2310_17556_b200 as fsb
from paper_2310_17556_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
prec = sys.argv[3] if len(sys.argv) > 3 else "f16x2"
dt = torch.float64 if (sys.argv[4] if len(sys.argv) > 4 else ("f64" if prec == "fp64" else "f32")) == "f64" \
    else torch.float32
dev = torch.device("cuda", 0)
S = torch.randn(n, m, device=dev, dtype=dt) / n ** 0.5
v = torch.randn(m, device=dev, dtype=dt)
system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
ctx = _lib.context_for(0, n, m)
ctx.profile(True)
for _ in range(3):
    sol = fsb.solve_chol(system, precision=prec)
torch.cuda.synchronize()
st = ctx.stage_ms()
print(f"n={n} m={m} {prec} {dt}: " + ", ".join(f"{k} {v:.3f}" for k, v in st.items() if v > 0)
      + f" | sum {sum(st.values()):.3f} ms, rel_residual {sol.rel_residual:.2e}")
