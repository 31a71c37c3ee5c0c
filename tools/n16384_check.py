"""BASELINE configs[4] per-rank workload on one GPU: n = 16384 with the column shard one of 8 ranks
owns (m_k = 1e7 / 8 = 1.25e6, fp32, S_k = 82 GB), through distributed.sharded_solve_chol_fused
on a 1-rank NCCL group (the all-reduce is then a no-op copy). A smaller m first cross-checks
f16x2 against the exact fp64 mode at n = 16384."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
import torch, torch.distributed as dist
from paper_2310_17556_b200 import distributed as fsd

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
dev = torch.device("cuda", 0)
n = 16384


def run(m, prec, dt, reps=2):
    g = torch.Generator(device=dev).manual_seed(m)     # same fp32 draws for every mode
    S = torch.empty(n, m, device=dev).normal_(generator=g).div_(n ** 0.5).to(dt)   # in place: S_k is 82 GB
    v = torch.randn(m, device=dev, generator=g).to(dt)
    torch.cuda.empty_cache()
    sol = fsd.sharded_solve_chol_fused(S, v, 1e-3, precision=prec)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        sol = fsd.sharded_solve_chol_fused(S, v, 1e-3, precision=prec)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"n={n} m={m} {prec}: {ms:.1f} ms  rel_residual {sol.rel_residual:.3e}  "
          f"SYRK-equivalent {n * n * m / (ms * 1e-3) / 1e12:.0f} TF/s", flush=True)
    x = sol.x_local.clone()
    del S, v, sol
    torch.cuda.empty_cache()
    return x


m_small = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
xa = run(m_small, "f16x2", torch.float32)
xb = run(m_small, "fp64", torch.float64, reps=1)
print(f"  f16x2 vs fp64 relerr(x) {((xa - xb).norm() / xb.norm()).item():.3e}", flush=True)
del xa, xb
from paper_2310_17556_b200 import _lib
_lib.release_contexts()
torch.cuda.empty_cache()
if len(sys.argv) <= 2 or sys.argv[2] != "small":
    run(1_250_000, "f16x2", torch.float32)
dist.destroy_process_group()
