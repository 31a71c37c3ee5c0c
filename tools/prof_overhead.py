"""Host overhead per solve: wall time vs device time (events) vs the sum of stage times."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2310_17556_b200 as fsb
from paper_2310_17556_b200 import _lib
n, m = 1024, 1_000_000
dev = torch.device("cuda", 0)
S = torch.randn(n, m, device=dev) / 32
v = torch.randn(m, device=dev)
system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
ctx = _lib.context_for(0, n, m)
ctx.profile(True)
for _ in range(3):
    fsb.solve_chol(system)
torch.cuda.synchronize()
walls, stages = [], []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
for _ in range(10):
    t1 = time.perf_counter()
    fsb.solve_chol(system)
    walls.append(time.perf_counter() - t1)
    stages.append(sum(ctx.stage_ms().values()))
e1.record(); torch.cuda.synchronize()
print(f"device per solve {e0.elapsed_time(e1) / 10:.3f} ms, wall per solve {1e3 * sum(walls) / 10:.3f} ms, "
      f"stage sum {sum(stages) / 10:.3f} ms")
ctx.profile(False)
e0.record()
for _ in range(10):
    fsb.solve_chol(system)
e1.record(); torch.cuda.synchronize()
print(f"profiling off: device per solve {e0.elapsed_time(e1) / 10:.3f} ms")
t1 = time.perf_counter()
for _ in range(100):
    fsb.solve_chol.__wrapped__ if hasattr(fsb.solve_chol, "__wrapped__") else None
