"""Fused last z-space step (FS_ZFUSE, default on) vs the full pass: solve time, the stored
residual vs an exact recompute (fsb.residual: y = S x with exact fp64 products), x agreement.

    FS_ZFUSE=1 python tools/zfuse_check.py run a.npz [n m]
    FS_ZFUSE=0 python tools/zfuse_check.py run b.npz [n m]
    python tools/zfuse_check.py compare a.npz b.npz
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def run(out, n, m):
    import torch
    import paper_2310_17556_b200 as fsb
    from paper_2310_17556_b200 import _lib
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(n + m)
    S = torch.randn(n, m, device=dev, generator=g) / n ** 0.5
    v = torch.randn(m, device=dev, generator=g)
    system = fsb.DampedSystem(fsb.ScoreMatrix(S), 1e-3, v)
    ctx = _lib.context_for(0, n, m)
    ctx.profile(True)
    sol = fsb.solve_chol(system)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        sol = fsb.solve_chol(system)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    st = ctx.stage_ms()
    a, r = fsb.residual(system, sol.x)
    info = {"zfuse": os.environ.get("FS_ZFUSE", "1"), "n": n, "m": m, "ms_median": float(np.median(ts)),
            "ms_min": float(min(ts)), "rel_residual": sol.rel_residual, "recomputed_rel_residual": r,
            "abs_residual": sol.abs_residual, "recomputed_abs_residual": a, "precision": sol.precision,
            "stage_ms": {k: round(x, 3) for k, x in st.items()}}
    print(json.dumps(info), flush=True)
    np.savez(out, x=sol.x.cpu().numpy(), info=np.frombuffer(json.dumps(info).encode(), dtype=np.uint8))


def compare(a, b):
    A, B = np.load(a), np.load(b)
    ia, ib = json.loads(A["info"].tobytes()), json.loads(B["info"].tobytes())
    xa, xb = A["x"], B["x"]
    print(json.dumps({"x_relerr": float(np.linalg.norm(xa - xb) / np.linalg.norm(xb)),
                      "ms": [ia["ms_median"], ib["ms_median"]],
                      "rel_residual": [ia["rel_residual"], ib["rel_residual"]],
                      "recomputed": [ia["recomputed_rel_residual"], ib["recomputed_rel_residual"]]}))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        n = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
        m = int(sys.argv[4]) if len(sys.argv) > 4 else 1_000_000
        run(sys.argv[2], n, m)
    else:
        compare(sys.argv[2], sys.argv[3])
