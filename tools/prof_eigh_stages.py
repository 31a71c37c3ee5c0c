"""Stage times of the eigh route at the headline (fs_eigh_solve profiling marks: gram, gemv_sv,
eig (potrf slot), eig_apply (trsv slot), x pass, residual, refine)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2310_17556_b200 as fsb
from paper_2310_17556_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
dev = torch.device("cuda", 0)
S = torch.randn(n, m, device=dev) / n ** 0.5
v = torch.randn(m, device=dev)
system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
ctx = _lib.context_for(0, n, m)
ctx.profile(True)
for prec in ("f16x2", "fp64"):
    for _ in range(3):
        sol = fsb.solve_svd_eigh(system, precision=prec)
        torch.cuda.synchronize()
    print(prec, {k: round(x, 3) for k, x in ctx.stage_ms().items()}, "sum", round(sum(ctx.stage_ms().values()), 3),
          "rel_res", sol.rel_residual, flush=True)
