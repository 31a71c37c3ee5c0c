"""Hypothesis property tests on the GPU path — the counterparts of the reference's own property
tests (pkg/tests/test_solvers.py:83-96 residual property, test_core.py:118-135 positive
definiteness for any damping) plus properties the GPU kernels must keep on their own:

  * solve_chol satisfies the original system: abs_residual <= 1e-8 ||v|| (fp64 scores, the
    reference's test) and the drop-in promise rel_residual <= 1e-8 for float32 scores
  * gram(S, lam) is exactly symmetric and its smallest eigenvalue >= lam - 1e-9 max|W|
  * power-of-two scaling: gram_packed(2^k S, 4^k lam) == 4^k gram_packed(S, lam) BIT FOR BIT in
    every precision (the F16X2 row scales are powers of two chosen from the row maxima, so the
    hi/lo planes, the tensor-core products and the fixed-order reductions are identical)
  * linearity in v of the fp64 solve, and agreement of the chol / eigh / svd routes

Shapes are small (the oracle-free properties need no CPU reference); every example runs the
CUDA kernels (the product path has no CPU fallback).
"""

import numpy as np
import pytest
import torch
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

pytestmark = pytest.mark.gpu

SETTINGS = dict(deadline=None, suppress_health_check=[HealthCheck.function_scoped_fixture])


@pytest.fixture(scope="module")
def fsb():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2310_17556_b200 as fsb
    return fsb


def rng_for(seed):
    return np.random.Generator(np.random.PCG64(seed))


def random_system(fsb, seed, n, m, lam, dtype=np.float64):
    rng = rng_for(seed)
    S = (rng.standard_normal((n, m)) / np.sqrt(n)).astype(dtype)
    v = rng.standard_normal(m).astype(dtype)
    return fsb.DampedSystem(fsb.ScoreMatrix(S), lam, v), S, v


@given(n=st.sampled_from([1, 2, 4, 8, 16, 33, 130]), m=st.integers(1, 400),
       lam=st.sampled_from([1e-6, 1e-3, 1.0, 10.0]), seed=st.integers(0, 9))
@settings(max_examples=60, **SETTINGS)
def test_residual_property(fsb, n, m, lam, seed):
    """test_solvers.py:83-96 on the GPU solve (fp64 scores: the reference's arithmetic)."""
    m = max(m, n)
    system, S, v = random_system(fsb, seed, n, m, lam)
    sol = fsb.solve_chol(system)
    assert sol.abs_residual <= 1e-8 * np.linalg.norm(v), (sol.abs_residual, np.linalg.norm(v))
    # the stored residual is the recomputed one (test_solvers.py:75-81)
    assert fsb.residual(system, sol.x, fsb.Variant.PLAIN) == (sol.abs_residual, sol.rel_residual)


@given(n=st.sampled_from([1, 3, 64, 65, 200]), m=st.integers(1, 3000),
       lam=st.sampled_from([1e-4, 1e-2, 1.0]), seed=st.integers(0, 99))
@settings(max_examples=40, **SETTINGS)
def test_float32_default_meets_promise(fsb, n, m, lam, seed):
    """float32 scores through the drop-in default (F16X2 + z-space refinement, fp64 recompute as
    the last resort): the reference's promise rel_residual <= 1e-8 (solvers.py:41-42)."""
    m = max(m, n)
    system, S, v = random_system(fsb, seed, n, m, lam, np.float32)
    sol = fsb.solve_chol(system)
    assert sol.rel_residual <= 1e-8, (sol.precision, sol.rel_residual)
    # the stored residual is that of the returned x (an exact recompute: y = S x, fp64 products; at the rounding floor
    # the summation order moves it by a few percent at most)
    _, rel = fsb.residual(system, sol.x, fsb.Variant.PLAIN)
    assert abs(sol.rel_residual - rel) <= 0.05 * rel + 1e-15, (sol.rel_residual, rel)


@given(n=st.integers(1, 32), m=st.integers(1, 48), lam_exp=st.integers(-6, 1), seed=st.integers(0, 2**32 - 1))
@settings(max_examples=60, **SETTINGS)
def test_positive_definite_for_any_damping(fsb, n, m, lam_exp, seed):
    """test_core.py:118-135 on the GPU Gram."""
    lam = 10.0 ** lam_exp
    S = fsb.ScoreMatrix(rng_for(seed).standard_normal((n, m)))
    W = fsb.gram(S, lam)
    assert np.array_equal(W, W.T)
    smallest = np.linalg.eigvalsh(W)[0]
    assert smallest >= lam - 1e-9 * max(1.0, np.abs(W).max())


@given(n=st.sampled_from([1, 5, 128, 129, 300]), m=st.integers(1, 20000), k=st.integers(-20, 20),
       prec=st.sampled_from(["f16x2", "tf32x3", "fp64"]), seed=st.integers(0, 99))
@settings(max_examples=40, **SETTINGS)
def test_gram_power_of_two_scaling_is_exact(fsb, n, m, k, prec, seed):
    rng = rng_for(seed)
    S = (rng.standard_normal((n, m)) * rng.uniform(0.1, 10.0, size=(n, 1))).astype(np.float32)
    dev = torch.device("cuda", 0)
    lam = 1e-3
    G1 = fsb.gram_packed(fsb.ScoreMatrix(torch.from_numpy(S).to(dev)), lam, prec).cpu().numpy()
    S2 = np.ldexp(S, k).astype(np.float32)
    G2 = fsb.gram_packed(fsb.ScoreMatrix(torch.from_numpy(S2).to(dev)), lam * 4.0 ** k, prec).cpu().numpy()
    assert np.array_equal(G2, np.ldexp(G1, 2 * k)), (prec, k, np.abs(G2 - np.ldexp(G1, 2 * k)).max())


@given(n=st.sampled_from([2, 17, 64, 257]), m=st.integers(300, 5000), seed=st.integers(0, 99),
       a=st.floats(-4, 4), b=st.floats(-4, 4))
@settings(max_examples=30, **SETTINGS)
def test_fp64_solve_is_linear_in_v(fsb, n, m, seed, a, b):
    rng = rng_for(seed)
    S = fsb.ScoreMatrix(rng.standard_normal((n, m)) / np.sqrt(n))
    v1, v2 = rng.standard_normal(m), rng.standard_normal(m)
    lam = 1e-3
    x1 = fsb.solve_chol(fsb.DampedSystem(S, lam, v1)).x
    x2 = fsb.solve_chol(fsb.DampedSystem(S, lam, v2)).x
    x12 = fsb.solve_chol(fsb.DampedSystem(S, lam, a * v1 + b * v2)).x
    ref = a * x1 + b * x2
    assert np.linalg.norm(x12 - ref) <= 1e-10 * max(1e-300, np.linalg.norm(x12) + abs(a) * np.linalg.norm(x1)
                                                    + abs(b) * np.linalg.norm(x2))


@given(n=st.sampled_from([1, 3, 32, 100, 160]), m=st.integers(1, 4000),
       lam=st.sampled_from([1e-4, 1e-2, 1.0]), seed=st.integers(0, 99))
@settings(max_examples=30, **SETTINGS)
def test_routes_agree(fsb, n, m, lam, seed):
    """chol, eigh (block / scalar Jacobi) and svd (Gram fast path or CholeskyQR3 + Jacobi SVD)
    solve the same full-rank system: x agrees to 1e-8 (fp64 scores, n <= m)."""
    m = max(m, n)
    system, S, v = random_system(fsb, seed, n, m, lam)
    xc = fsb.solve_chol(system).x
    xe = fsb.solve_svd_eigh(system).x
    xs = fsb.solve_svd_direct(system).x
    nc = np.linalg.norm(xc)
    assert np.linalg.norm(xe - xc) <= 1e-8 * nc and np.linalg.norm(xs - xc) <= 1e-8 * nc
