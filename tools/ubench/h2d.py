"""H2D bandwidth: pinned contiguous vs pinned 2-D column chunks (cudaMemcpy2DAsync via torch)."""
import torch, time
n, m = 1024, 1_000_000
h = torch.empty(n, m, dtype=torch.float32, pin_memory=True); h.normal_()
d = torch.empty(n, m, dtype=torch.float32, device="cuda")
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize()
    print("contiguous 4.1 GB: %.1f ms  %.1f GB/s" % (e0.elapsed_time(e1), 4.096e9 / e0.elapsed_time(e1) / 1e6))
for cw in (131072, 250000):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for a in range(0, m, cw):
        b = min(m, a + cw)
        d[:, a:b].copy_(h[:, a:b], non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print("2-D chunks of %d cols: %.1f ms  %.1f GB/s" % (cw, e0.elapsed_time(e1), 4.096e9 / e0.elapsed_time(e1) / 1e6))
