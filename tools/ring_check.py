"""F16X2 ring SYRK vs the pre-tiled path (FS_F16_RING=0): Gram bits, solve parity, stage times.

    FS_F16_RING=1 python tools/ring_check.py run ring.npz
    FS_F16_RING=0 python tools/ring_check.py run tiled.npz
    python tools/ring_check.py compare ring.npz tiled.npz
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

SHAPES = [(128, 70000), (256, 200000), (300, 65536 + 37), (512, 300000), (1000, 100003), (1024, 1_000_000),
          (2048, 400000), (2816, 200000), (64, 4096)]


def run(out):
    import torch
    import paper_2310_17556_b200 as fsb
    from paper_2310_17556_b200 import _lib
    from oracle import fisher_oracle as O
    dev = torch.device("cuda", 0)
    res = {}
    for n, m in SHAPES:
        g = torch.Generator(device=dev).manual_seed(n * 7 + m)
        S = torch.randn(n, m, device=dev, generator=g) / n ** 0.5
        v = torch.randn(m, device=dev, generator=g)
        sm = fsb.ScoreMatrix(S)
        G = fsb.gram_packed(sm, 1e-3, precision="f16x2").cpu().numpy()
        system = fsb.DampedSystem(sm, 1e-3, v)
        ctx = _lib.context_for(0, n, m)
        ctx.profile(True)
        sol = fsb.solve_chol(system, precision="f16x2", refine=0)
        torch.cuda.synchronize()
        ts, gs = [], []
        for _ in range(5):
            t0 = time.perf_counter()
            sol = fsb.solve_chol(system, precision="f16x2", refine=0)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
            st = ctx.stage_ms()
            gs.append(st["gram"] + st["gemv_sv"])
        x = sol.x.cpu().numpy() if hasattr(sol.x, "cpu") else np.asarray(sol.x)
        key = f"{n}x{m}"
        res[key + "_G"] = G
        res[key + "_x"] = x
        # oracle parity on the small shapes (fp64 solve of the identical fp32 system)
        err = None
        if n * m <= 3e7:
            S64 = S.double().cpu().numpy()
            ref = O.solve_chol(S64, v.double().cpu().numpy(), 1e-3)
            err = float(O.rel_err(x, ref.x))
        info = {"n": n, "m": m, "solve_ms": float(np.median(ts)), "gram_u_ms": float(np.median(gs)),
                "rel_residual": float(sol.rel_residual), "relerr_vs_oracle": err}
        print(json.dumps(info), flush=True)
        res[key + "_info"] = np.frombuffer(json.dumps(info).encode(), dtype=np.uint8)
        del S, sm, system
        torch.cuda.empty_cache()
    np.savez(out, **res)


def compare(a, b):
    A, B = np.load(a), np.load(b)
    for n, m in SHAPES:
        key = f"{n}x{m}"
        if key + "_G" not in A or key + "_G" not in B:
            continue
        ga, gb = A[key + "_G"], B[key + "_G"]
        xa, xb = A[key + "_x"], B[key + "_x"]
        ia = json.loads(A[key + "_info"].tobytes()); ib = json.loads(B[key + "_info"].tobytes())
        print(f"{key}: G bit-identical {np.array_equal(ga, gb)} (max rel diff "
              f"{np.abs(ga - gb).max() / np.abs(gb).max():.2e}), x relerr {np.linalg.norm(xa - xb) / np.linalg.norm(xb):.2e}, "
              f"gram+u {ia['gram_u_ms']:.3f} vs {ib['gram_u_ms']:.3f} ms, solve {ia['solve_ms']:.3f} vs {ib['solve_ms']:.3f} ms, "
              f"oracle relerr {ia['relerr_vs_oracle']} / {ib['relerr_vs_oracle']}")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        compare(sys.argv[2], sys.argv[3])
