import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from oracle import fisher_oracle as O
import paper_2310_17556_b200 as fsb
S, v, lam = O.generate_problem(41, 256, 65536, 1e-3)
S32, v32 = S.astype(np.float32), v.astype(np.float32)
system = fsb.DampedSystem(fsb.ScoreMatrix(S32), lam, v32)
ref = O.solve_chol(S32.astype(np.float64), v32.astype(np.float64), lam)
for prec in ("f16x2", "tf32x3", "fp64"):
    out = []
    for k in (0, 1, 2, 3, 4, 6, 8, 12):
        sol = fsb.solve_chol(system, precision=prec, refine=k)
        out.append(f"{k}:{sol.rel_residual:.2e}/{O.rel_err(sol.x, ref.x):.1e}")
    print(prec, " ".join(out))
