"""Launch the Gram stage alone (for ncu isolation): fs_gram_packed at the headline shape."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17556_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
prec = sys.argv[3] if len(sys.argv) > 3 else "tf32x3"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
dev = torch.device("cuda", 0)
dt = torch.float64 if prec == "fp64" else torch.float32
S = torch.randn(n, m, device=dev, dtype=dt) / n ** 0.5
G = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device=dev)
ctx = _lib.context_for(0, n, m)
st = torch.cuda.current_stream().cuda_stream
P = {"tf32x3": _lib.FS_PREC_TF32X3, "f16x2": _lib.FS_PREC_F16X2, "fp64": _lib.FS_PREC_FP64}[prec]
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(reps):
    e0.record()
    rc = ctx.lib.fs_gram_packed(ctx.handle, _lib.FS_F32 if dt == torch.float32 else _lib.FS_F64, P, S.data_ptr(),
                                n, m, m, 0.0, G.data_ptr(), st)
    e1.record()
    torch.cuda.synchronize()
    assert rc == 0, ctx.last_error()
    print(f"gram {prec} n={n} m={m}: {e0.elapsed_time(e1):.3f} ms  "
          f"{n * (n + 1) * m / e0.elapsed_time(e1) / 1e9:.1f} TF/s")
