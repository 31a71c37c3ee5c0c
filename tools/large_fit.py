"""Large-n evidence on one B200.

  1. potrf (+ both fused TRSVs) stage time for n = 1024 ... 16384 (fs_potrf on a damped random
     Gram, CUDA events, n^3/3 flop).
  2. n = 16384, m = 2e6 fp32 scores (131 GB) solved in F16X2 on ONE GPU: the tiled copy is capped
     (K-chunked Gram), so S + at most 16 GB of planes fit.  Stage times + the exact fp64 residual.

    python tools/large_fit.py [--skip-solve] [--m 2000000]
"""
import argparse
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2310_17556_b200 as fsb
from paper_2310_17556_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--skip-solve", action="store_true")
ap.add_argument("--m", type=int, default=2_000_000)
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--potrf-ns", default="1024,2048,4096,8192,16384")
args = ap.parse_args()
dev = torch.device("cuda", 0)
out = {"potrf": [], "solve": None}

for n in [int(x) for x in args.potrf_ns.split(",") if x]:
    A = torch.randn(n, n + 64, device=dev, dtype=torch.float64)
    W0 = (A @ A.T) / n + 1e-3 * torch.eye(n, device=dev, dtype=torch.float64)
    del A
    ctx = _lib.context_for(0, n, 8)
    st = torch.cuda.current_stream().cuda_stream
    ts = []
    for rep in range(3):
        W = torch.tril(W0).contiguous()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        piv = ctypes.c_int64(-1)
        e0.record()
        rc = ctx.lib.fs_potrf(ctx.handle, W.data_ptr(), n, n, ctypes.byref(piv), st)
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0, (n, rc)
        ts.append(e0.elapsed_time(e1))
    err = float((W @ W.T - W0).abs().max() / W0.abs().max())
    ms = min(ts)
    rec = {"n": n, "ms": round(ms, 3), "TFLOPs": round(n ** 3 / 3 / (ms * 1e-3) / 1e12, 2), "max_rel_LLt_err": err}
    out["potrf"].append(rec)
    print(json.dumps(rec), flush=True)
    del W, W0
    torch.cuda.empty_cache()

if not args.skip_solve:
    n, m = args.n, args.m
    g = torch.Generator(device=dev).manual_seed(16384)
    S = torch.empty(n, m, device=dev).normal_(generator=g).div_(n ** 0.5)   # in place: n m 4 bytes
    v = torch.randn(m, device=dev, generator=g)
    sm = fsb.ScoreMatrix._owned(S)            # no private copy (S alone is 131 GB at the default)
    system = fsb.DampedSystem(sm, 1e-3, v)
    ctx = _lib.context_for(0, n, m)
    ctx.profile(True)
    sol = fsb.solve_chol(system, precision="f16x2")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sol = fsb.solve_chol(system, precision="f16x2")
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    rec = {"n": n, "m": m, "precision": "f16x2", "refine": "auto", "ms": round(ms, 1),
           "rel_residual": sol.rel_residual, "stage_ms": {k: round(v, 2) for k, v in ctx.stage_ms().items()},
           "peak_mem_GB": round(torch.cuda.max_memory_allocated() / 1e9, 1),
           "gram_TFLOPs": None}
    g_ms = rec["stage_ms"]["gram"] + rec["stage_ms"]["gemv_sv"]
    rec["gram_TFLOPs"] = round(n * (n + 1) * m / (g_ms * 1e-3) / 1e12, 1)
    out["solve"] = rec
    print(json.dumps(rec), flush=True)
print(json.dumps(out))
