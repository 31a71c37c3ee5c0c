"""Factor a damped Gram matrix of the headline shape (n=1024) for ncu launch lists."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17556_b200 import _lib
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
dev = torch.device("cuda", 0)
A = torch.randn(n, 2 * n, device=dev, dtype=torch.float64)
W0 = (A @ A.T) / n + torch.eye(n, device=dev, dtype=torch.float64)
ctx = _lib.context_for(0, n, 8)
st = torch.cuda.current_stream().cuda_stream
for rep in range(3):
    W = torch.tril(W0).contiguous()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    piv = ctypes.c_int64(-1)
    e0.record()
    rc = ctx.lib.fs_potrf(ctx.handle, W.data_ptr(), n, n, ctypes.byref(piv), st)
    e1.record(); torch.cuda.synchronize()
    print(f"potrf n={n}: {e0.elapsed_time(e1):.3f} ms rc={rc}")
L = W
print("max |LL^T - W|/|W| =", float((L @ L.T - W0).abs().max() / W0.abs().max()))
