"""Break the e2e (host numpy -> numpy x) solve into host-side and device-stage times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2310_17556_b200 as fsb
from paper_2310_17556_b200 import _lib

n, m = 1024, 1_000_000
S = torch.empty((n, m), dtype=torch.float32, pin_memory=True)
S.normal_().mul_(n ** -0.5)
v = torch.empty(m, dtype=torch.float32, pin_memory=True).normal_()
Sh, vh = S.numpy(), v.numpy()
ctx = _lib.context_for(0, n, m)
ctx.profile(True)
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    system = fsb.DampedSystem(fsb.ScoreMatrix(Sh), 1e-3, vh)
    t1 = time.perf_counter()
    sol = fsb.solve_chol(system)
    t2 = time.perf_counter()
    st = ctx.stage_ms()
    print(f"construct {1e3*(t1-t0):.2f} ms  solve_chol {1e3*(t2-t1):.2f} ms  stages "
          + " ".join(f"{k}={v:.2f}" for k, v in st.items()) + f"  sum={sum(st.values()):.2f}")
