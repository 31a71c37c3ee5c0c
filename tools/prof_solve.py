"""One headline-shape solve_chol on device tensors (for ncu isolation of a stage kernel)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2310_17556_b200 as fsb

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
dev = torch.device("cuda", 0)
S = torch.randn(n, m, device=dev, dtype=torch.float32) / n ** 0.5
v = torch.randn(m, device=dev, dtype=torch.float32)
system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
for _ in range(reps):
    sol = fsb.solve_chol(system, precision=os.environ.get("FS_PREC", "auto"))
    torch.cuda.synchronize()
print("rel_residual", sol.rel_residual)
