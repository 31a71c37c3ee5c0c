"""Time the SYRK alone (fs_chol_solve's Gram stage via the profiling events) at the headline shape."""
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
del S
ctx = _lib.context_for(0, n, m); ctx.profile(True)
g = []
for i in range(4):
    try:   # ablated kernels produce garbage Grams: a failed factorization still records the stage times
        fsb.solve_chol(system, precision=os.environ.get("FS_PREC", "f16x2"), diagnostics=False, refine=False)
    except fsb.FactorizationError:
        pass
    g.append(ctx.stage_ms())
print("gram %.3f ms  gemv_sv+retile %.3f ms" % (min(x["gram"] for x in g[1:]), min(x["gemv_sv"] for x in g[1:])))
