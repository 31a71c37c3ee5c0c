"""One solve_svd_direct at the headline shape (device fp32 scores) for an ncu launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2310_17556_b200 as fsb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
dev = torch.device("cuda", 0)
S = torch.randn(n, m, device=dev) / n ** 0.5
v = torch.randn(m, device=dev)
system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
sol = fsb.solve_svd_direct(system)
torch.cuda.synchronize()
print("rel_residual", sol.rel_residual)
