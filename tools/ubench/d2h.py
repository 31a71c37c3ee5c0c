"""D2H of an 8 MB fp64 vector: pageable fresh numpy vs pinned staging (+ host copy)."""
import time
import numpy as np
import torch
m = 1_000_000
d = torch.randn(m, dtype=torch.float64, device="cuda")
pin = torch.empty(m, dtype=torch.float64, pin_memory=True)
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    x = np.empty(m); torch.from_numpy(x).copy_(d)
    t1 = time.perf_counter()
    pin.copy_(d); torch.cuda.synchronize()
    t2 = time.perf_counter()
    y = pin.numpy().copy()
    t3 = time.perf_counter()
    z = np.empty(m); z[:] = 0
    t4 = time.perf_counter()
    print(f"pageable fresh {1e3*(t1-t0):.3f} ms | pinned d2h {1e3*(t2-t1):.3f} ms + host copy {1e3*(t3-t2):.3f} ms | prefault {1e3*(t4-t3):.3f} ms")
