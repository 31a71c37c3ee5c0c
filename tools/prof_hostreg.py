"""Why pageable uploads are staged instead of pinned in place: cudaHostRegister of the caller's
4.1 GB numpy array costs ~350-390 ms (+70-130 ms to unregister) before a 74 ms DMA, against ~105 ms
for the 8-worker staging ring (tools/prof_pageable.py)."""
import time, numpy as np, torch
S = np.random.default_rng(0).standard_normal((1024, 1_000_000), dtype=np.float32)
dst = torch.empty((1024, 1_000_000), dtype=torch.float32, device="cuda")
import torch.cuda
rt = torch.cuda.cudart()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = rt.cudaHostRegister(S.ctypes.data, S.nbytes, 0)
    t1 = time.perf_counter()
    src = torch.from_numpy(S)
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    rt.cudaHostUnregister(S.ctypes.data)
    t3 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.1f} ms (rc {r}), copy {1e3*(t2-t1):.1f} ms, unregister {1e3*(t3-t2):.1f} ms", flush=True)
