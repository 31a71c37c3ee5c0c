"""One small invocation of every hand-written kernel family, for compute-sanitizer
(tools/sanitize.sh runs it under memcheck, racecheck and synccheck).

    python tools/sanitize_driver.py [stage ...]     stages: gram16 gram32 gram64 chol eigh svd apply multi
"""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np
import torch

import paper_2310_17556_b200 as fsb
from paper_2310_17556_b200 import solvers as fs_solvers

stages = sys.argv[1:] or ["gram16", "gram32", "gram64", "chol", "eigh", "svd", "apply"]
dev = torch.device("cuda", 0)
rng = np.random.Generator(np.random.PCG64(0))
n, m = 256, 8192
S = (rng.standard_normal((n, m)) / np.sqrt(n)).astype(np.float32)
v = rng.standard_normal(m).astype(np.float32)
St = torch.from_numpy(S).to(dev)
vt = torch.from_numpy(v).to(dev)
sm = fsb.ScoreMatrix(St)
for stage in stages:
    if stage == "gram16":      # syrk_tc<f16> (tcgen05 cta_group::2, bulk copies, mbarriers) + retile16
        fsb.gram_packed(sm, 1e-3, precision="f16x2")
    elif stage == "gram32":    # syrk_tc<tf32>
        fsb.gram_packed(sm, 1e-3, precision="tf32x3")
    elif stage == "gram64":    # syrk_dmma
        fsb.gram_packed(sm, 1e-3, precision="fp64")
    elif stage == "chol":      # retile16 + SYRK + potrf_persistent (grid barriers) + cols_solve_y_cl (DSMEM st.async) + residual
        system = fsb.DampedSystem(sm, 1e-3, vt)
        fsb.solve_chol(system, precision="f16x2", refine=2)
        fsb.solve_chol(system, precision="fp64")
    elif stage == "eigh":      # Jacobi eigensolver (cooperative grid barriers)
        fsb.solve_svd_eigh(fsb.DampedSystem(fsb.ScoreMatrix(St[:64, :2048].contiguous()), 1e-3, vt[:2048]),
                           precision="fp64")
    elif stage == "svd":       # CholeskyQR3 (apply_rows, tri_inverse) + one-sided Jacobi SVD
        fsb.thin_svd_direct(fsb.ScoreMatrix(St[:64, :2048].double().contiguous()))
    elif stage == "apply":
        T = torch.from_numpy(rng.standard_normal((130, n))).to(dev)
        fs_solvers._apply_rows(T, sm.tensor)
    torch.cuda.synchronize()
    print("stage ok:", stage, flush=True)
