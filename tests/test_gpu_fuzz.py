"""Randomised shapes through the whole drop-in solve (every precision), against the CPU oracle:
odd n and m, partial 64-row blocks, partial 128-row tile pairs, partial 64-column K-blocks and
256-byte panels, tiny and tall-ish shards — the edge cases of the cluster x + y pass, the TRSV
kernels (single CTA / cluster / flag-chained), the persistent and blocked potrf and the split-K
plans.  Tolerances as in SURVEY §8d (fp32 modes 1e-6, fp64 1e-10, relative to the fp64 solve of
the identical system)."""

import numpy as np
import pytest
import torch

from oracle import fisher_oracle as O

pytestmark = pytest.mark.gpu

_rng = np.random.Generator(np.random.PCG64(2026))
CASES = []
for i in range(24):
    n = int(_rng.choice([1, 2, 3, 63, 64, 65, 127, 129, 255, 257, 513, 1000, 1023, 1025, 1500, 2049]))
    m = int(max(n + 1, _rng.integers(2, 120_000)))
    prec = ["f16x2", "tf32x3", "fp64"][i % 3]
    CASES.append((i, n, m, prec))


@pytest.fixture(scope="module")
def fsb():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2310_17556_b200 as fsb
    return fsb


@pytest.mark.parametrize("case,n,m,prec", CASES)
def test_random_shape_solve(fsb, case, n, m, prec):
    S, v, lam = O.generate_problem(1000 + case, n, m, float(_rng.choice([1e-3, 1e-1, 1.0])))
    dt = np.float64 if prec == "fp64" and case % 2 else np.float32
    S, v = S.astype(dt), v.astype(dt)
    dev = torch.device("cuda", 0)
    system = fsb.DampedSystem(fsb.ScoreMatrix(torch.from_numpy(S).to(dev)), lam, torch.from_numpy(v).to(dev))
    sol = fsb.solve_chol(system, precision=prec)
    ref = O.solve_chol(S.astype(np.float64), v.astype(np.float64), lam)
    x = sol.x.cpu().numpy()
    # the drop-in default refines to the reference's rule in every mode, so x is fp64-accurate
    assert O.rel_err(x, ref.x) <= 1e-8, (n, m, prec, O.rel_err(x, ref.x))
    assert sol.rel_residual <= 1e-8, sol.rel_residual
