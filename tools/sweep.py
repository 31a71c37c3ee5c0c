"""BASELINE configs[2]/[3] sweeps: solve_chol device ms over n (m = 1e6) and over m (n = 1024).

Device-resident N(0,1)/sqrt(n) scores, lambda = 1e-3; per point 2 untimed + `reps` timed solves
(CUDA events on the current stream, inputs > L2). Writes one JSON document (argv[1], default
gpurun_out/sweep.json) — the committed copy is profiles/r01_sweep.json.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2310_17556_b200 as fsb


def point(n, m, precision, reps=3):
    dev = torch.device("cuda", 0)
    dt = torch.float64 if precision == "fp64" else torch.float32
    g = torch.Generator(device=dev).manual_seed(n * 7 + m)
    S = torch.randn(n, m, device=dev, dtype=dt, generator=g) / n ** 0.5
    v = torch.randn(m, device=dev, dtype=dt, generator=g)
    system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
    for _ in range(2):
        sol = fsb.solve_chol(system, precision=precision)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        sol = fsb.solve_chol(system, precision=precision)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = float(n) * n * m          # lower-triangle SYRK (n(n+1)/2 x m x 2)
    out = {"n": n, "m": m, "precision": precision, "ms": round(ms, 4),
           "rel_residual": float(sol.rel_residual),
           "s_gb": round(S.numel() * S.element_size() / 1e9, 3),
           "s_stream_gbps": round(S.numel() * S.element_size() / (ms * 1e-3) / 1e9, 1),
           "syrk_tflops_whole_solve": round(flops / (ms * 1e-3) / 1e12, 1)}
    del system, S, v, sol
    torch.cuda.empty_cache()
    return out


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep.json"
    pts = []
    # fp64 stops where S plus ScoreMatrix's private copy (2 x 8 n m bytes) would not fit in HBM
    plan = [(n, 1_000_000, "f16x2") for n in (256, 512, 1024, 2048, 4096, 8192)]
    plan += [(n, 1_000_000, "fp64") for n in (256, 512, 1024, 2048, 4096)]
    plan += [(1024, m, "f16x2") for m in (100_000, 300_000, 3_000_000, 10_000_000)]
    plan += [(1024, m, "fp64") for m in (100_000, 300_000, 3_000_000)]
    t0 = time.time()
    for n, m, p in plan:
        r = point(n, m, p)
        pts.append(r)
        print(json.dumps(r), flush=True)
    doc = {"device": torch.cuda.get_device_name(0), "lam": 1e-3, "data": "synthetic N(0,1)/sqrt(n)",
           "timing": "CUDA events, 2 warm-up + 3 timed solves per point, device-resident",
           "wall_s": round(time.time() - t0, 1), "points": pts}
    os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
