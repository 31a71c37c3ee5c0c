"""CPU oracle for the damped-Fisher Cholesky solve — TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference package's hot path
(``fisher_solve`` under /root/reference/pkg/src).  It exists so that the GPU
product can be checked against the reference algorithm on identical inputs.

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` leg may import this module.
  * The product package ``paper_2310_17556_b200`` never imports it: there is
    no CPU fallback on the product path.

Pinning: ``tests/golden/make_golden.py`` runs the *real* reference in the
survey container and commits its outputs (x, W, L, u, residuals) as fixtures;
``tests/test_oracle_golden.py`` checks this restatement against them.  The
reference's own arithmetic lives in numpy (OpenBLAS ``dsyrk``/``dgemv``) and
scipy (LAPACK ``dpotrf``/``dtrtrs``); the restatement calls the same routines
in the same order, so it agrees with the fixtures to round-off (bit-exact on
the machine that generated them).

Every function cites the reference file:line it follows; paths are relative
to /root/reference/pkg/src/fisher_solve/.
"""

from __future__ import annotations

from dataclasses import dataclass
from time import perf_counter

import numpy as np
from scipy.linalg import get_lapack_funcs, solve_triangular

EPS = float(np.finfo(np.float64).eps)          # core.py:16
REFINE_ABOVE_REL = 1e-10                        # solvers.py:43
DEFAULT_SIGMA_FLOOR = 1e-12                     # solvers.py:39
REL_RESIDUAL_GATE = 1e-6                        # bench.py:40


class OracleFactorizationError(RuntimeError):
    """Mirror of core.py:51-60 (FactorizationError with a 0-based pivot)."""

    def __init__(self, message, pivot=None):
        super().__init__(message)
        self.pivot = pivot


@dataclass
class OracleSolution:
    """Mirror of core.py:206-223 (Solution)."""

    x: np.ndarray
    abs_residual: float
    rel_residual: float
    wall_seconds: float
    refined: bool = False


def generate_problem(seed: int, n: int, m: int, lam: float = 1e-3):
    """Restates bench.py:127-171 for Kind.REAL_GAUSSIAN.

    PCG64(seed); S = standard_normal((n, m)) / sqrt(n) drawn first in
    row-major order (bench.py:155-159), then v = standard_normal(m)
    (bench.py:160).  Returns float64 (S, v, lam).
    """
    rng = np.random.Generator(np.random.PCG64(int(seed)))
    S = rng.standard_normal((int(n), int(m))) / np.sqrt(float(n))
    v = rng.standard_normal(int(m))
    return S, v, float(lam)


def random_system(seed: int, n: int, m: int, lam: float):
    """Restates tests/test_solvers.py:68-71 (the per-test generator)."""
    rng = np.random.Generator(np.random.PCG64(int(seed)))
    S = rng.standard_normal((n, m)) / np.sqrt(n)
    return S, rng.standard_normal(m), float(lam)


def gram(S: np.ndarray, lam: float) -> np.ndarray:
    """W = S S^T + lam I, symmetrized (core.py:270-290, real branch :284-289)."""
    A = np.ascontiguousarray(S, dtype=np.float64)
    W = A @ A.T                                  # core.py:284 (numpy -> dsyrk)
    W = 0.5 * (W + W.T)                          # core.py:287
    W[np.diag_indices(A.shape[0])] += lam        # core.py:289
    return W


def cholesky_lower(W: np.ndarray) -> np.ndarray:
    """LAPACK dpotrf(lower, clean) with the reference's pivot mapping (solvers.py:74-90)."""
    potrf, = get_lapack_funcs(("potrf",), (W,))
    L, info = potrf(W, lower=1, clean=1)          # solvers.py:80-81
    if info > 0:                                  # solvers.py:82-87
        raise OracleFactorizationError(
            f"Gram matrix is not positive definite at pivot {info - 1}", pivot=info - 1)
    if info < 0:                                  # solvers.py:88-89
        raise ValueError(f"invalid argument {-info} to LAPACK potrf")
    return L


def chol_apply(A: np.ndarray, lam: float, L: np.ndarray, b: np.ndarray) -> np.ndarray:
    """x = (b - A^T L^-T L^-1 A b) / lam, right to left (solvers.py:101-127, real)."""
    t1 = A @ b                                                                 # :110
    t2 = solve_triangular(L, t1, lower=True, trans="N", check_finite=False)   # :111
    t3 = solve_triangular(L, t2, lower=True, trans="T", check_finite=False)   # :114
    w = t3 @ A                                                                 # :122
    x = b - w                                                                  # :124
    x /= lam                                                                   # :126
    return x


def apply_operator(A: np.ndarray, lam: float, x: np.ndarray) -> np.ndarray:
    """(S^T S + lam I) x matrix-free, PLAIN variant (core.py:293-297)."""
    return (A @ x) @ A + lam * x


def residual(A: np.ndarray, lam: float, v: np.ndarray, x: np.ndarray):
    """(||Ax - v||, ||Ax - v|| / max(||v||, eps)) (core.py:307-322)."""
    r = apply_operator(A, lam, x) - v
    abs_res = float(np.linalg.norm(r))
    return abs_res, abs_res / max(float(np.linalg.norm(v)), EPS)


def solve_chol(S: np.ndarray, v: np.ndarray, lam: float, refine_above: float = REFINE_ABOVE_REL):
    """Restates _solve_chol_impl for Variant.PLAIN (solvers.py:151-206).

    gram -> potrf -> chol_apply -> first-pass residual; if rel > 1e-10 one
    correction pass with the same factor, then a fresh residual (solvers.py:183-194).
    """
    t0 = perf_counter()
    A = np.ascontiguousarray(S, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    L = cholesky_lower(gram(A, lam))                       # solvers.py:93-98
    x = chol_apply(A, lam, L, v)                           # :159
    r = apply_operator(A, lam, x)                          # :164
    np.subtract(r, v, out=r)                               # :168
    abs_res = float(np.linalg.norm(r))                     # :169
    rel_res = abs_res / max(float(np.linalg.norm(v)), EPS)  # :170
    if rel_res <= refine_above:                            # :171
        return OracleSolution(x, abs_res, rel_res, perf_counter() - t0, refined=False)
    np.negative(r, out=r)                                  # :186
    d = chol_apply(A, lam, L, r)                           # :187
    x += d                                                 # :188
    abs_res, rel_res = residual(A, lam, v, x)              # :192 -> _finish :139
    return OracleSolution(x, abs_res, rel_res, perf_counter() - t0, refined=True)


# ---------------------------------------------------------------- complex scores

def generate_problem_complex(seed: int, n: int, m: int, lam: float = 1e-3):
    """Restates bench.py:161-165 (Kind.COMPLEX_GAUSSIAN): PCG64(seed); the full real block, then
    the full imaginary block (row-major), S = (re + 1j im)/sqrt(n); v = normal(m) + 1j normal(m)."""
    rng = np.random.Generator(np.random.PCG64(int(seed)))
    re = rng.standard_normal((int(n), int(m)))
    im = rng.standard_normal((int(n), int(m)))
    S = (re + 1j * im) / np.sqrt(float(n))
    v = rng.standard_normal(int(m)) + 1j * rng.standard_normal(int(m))
    return S, v, float(lam)


def solve_chol_hermitian(S: np.ndarray, v: np.ndarray, lam: float, refine_above: float = REFINE_ABOVE_REL):
    """Restates _solve_chol_impl for Variant.HERMITIAN (solvers.py:151-213): W = S S^H + lam I
    symmetrised (core.py:280-290), complex potrf, x = (b - S^H L^-H L^-1 S b)/lam (solvers.py:101-127),
    residual of S^H S x + lam x - v (core.py:299-302), one refinement pass when rel > 1e-10."""
    t0 = perf_counter()
    A = np.ascontiguousarray(S, dtype=np.complex128)
    v = np.ascontiguousarray(v, dtype=np.complex128)
    W = A @ A.conj().T                                     # core.py:282
    W = 0.5 * (W + W.conj().T)                             # core.py:287
    W[np.diag_indices(A.shape[0])] += lam                  # core.py:289
    L = cholesky_lower(W)

    def apply(b):                                          # solvers.py:101-127, hermitian branch
        t1 = A @ b
        t2 = solve_triangular(L, t1, lower=True, trans="N", check_finite=False)
        t3 = solve_triangular(L, t2, lower=True, trans="C", check_finite=False)
        w = np.conj(np.conj(t3) @ A)
        return (b - w) / lam

    def op(x):                                             # core.py:299-302
        return np.conj(np.conj(A @ x) @ A) + lam * x

    x = apply(v)
    r = op(x) - v
    abs_res = float(np.linalg.norm(r))
    rel_res = abs_res / max(float(np.linalg.norm(v)), EPS)
    if rel_res <= refine_above:
        return OracleSolution(x, abs_res, rel_res, perf_counter() - t0, refined=False)
    x = x + apply(-r)                                      # solvers.py:186-188
    r = op(x) - v
    abs_res = float(np.linalg.norm(r))
    return OracleSolution(x, abs_res, abs_res / max(float(np.linalg.norm(v)), EPS), perf_counter() - t0,
                          refined=True)


def solve_realpart(S: np.ndarray, v: np.ndarray, lam: float):
    """Restates solve_realpart (solvers.py:216-240): C = [Re S; Im S] (sr.py:61-70), the plain route
    on C, residual of the REALPART operator (core.py:303-305) against the real v."""
    A = np.ascontiguousarray(S, dtype=np.complex128)
    C = np.concatenate([A.real, A.imag], axis=0)
    inner = solve_chol(C, np.asarray(v, dtype=np.float64), lam)
    re, im = A.real, A.imag
    r = (re @ inner.x) @ re + (im @ inner.x) @ im + lam * inner.x - v
    abs_res = float(np.linalg.norm(r))
    return OracleSolution(inner.x, abs_res, abs_res / max(float(np.linalg.norm(v)), EPS), inner.wall_seconds,
                          refined=inner.refined)


def thin_svd_eigh(S: np.ndarray, sigma_floor: float = DEFAULT_SIGMA_FLOOR):
    """Thin SVD from the Gram eigendecomposition (solvers.py:243-277, real)."""
    A = np.ascontiguousarray(S, dtype=np.float64)
    if A.shape[0] > A.shape[1]:
        raise ValueError("thin_svd_eigh requires n <= m")  # :255-256
    G = A @ A.T                                          # :258
    G = 0.5 * (G + G.T)                                  # :259
    evals, U = np.linalg.eigh(G)                         # :261 (dsyevd)
    evals = evals[::-1]                                  # :264
    U = U[:, ::-1]                                       # :265
    sigma = np.sqrt(np.clip(evals, 0.0, None))           # :266
    keep = sigma > sigma_floor * sigma[0]                # :267
    U = np.ascontiguousarray(U[:, keep])
    sigma = np.ascontiguousarray(sigma[keep])
    if sigma.size == 0:
        return U, sigma, np.zeros((A.shape[1], 0))       # :270-271
    V = A.T @ (U / sigma)                                # :272-276
    return U, sigma, V


def thin_svd_direct(S: np.ndarray):
    """Thin SVD via dgesdd, dropping exact zeros (solvers.py:280-291)."""
    U, s, Vh = np.linalg.svd(np.asarray(S, dtype=np.float64), full_matrices=False)
    keep = s > 0.0
    return np.ascontiguousarray(U[:, keep]), np.ascontiguousarray(s[keep]), Vh[keep].T


def solve_from_factors(sigma: np.ndarray, V: np.ndarray, lam: float, v: np.ndarray):
    """x = V (sigma^2+lam)^-1 V^T v + (v - V V^T v)/lam (solvers.py:318-326)."""
    v = np.asarray(v, dtype=np.float64)
    if sigma.size == 0:
        return v / lam                                   # :319
    t = v @ V                                            # :325
    return V @ (t / (sigma ** 2 + lam)) + (v - V @ t) / lam   # :326


def solve_svd_eigh(S, v, lam, sigma_floor=DEFAULT_SIGMA_FLOOR):
    """solvers.py:347-354 (residual against the source matrix, :327-330)."""
    t0 = perf_counter()
    _, sigma, V = thin_svd_eigh(S, sigma_floor)
    x = solve_from_factors(sigma, V, lam, v)
    a, r = residual(np.asarray(S, np.float64), lam, np.asarray(v, np.float64), x)
    return OracleSolution(x, a, r, perf_counter() - t0)


def solve_svd_direct(S, v, lam):
    """solvers.py:357-364."""
    t0 = perf_counter()
    _, sigma, V = thin_svd_direct(S)
    x = solve_from_factors(sigma, V, lam, v)
    a, r = residual(np.asarray(S, np.float64), lam, np.asarray(v, np.float64), x)
    return OracleSolution(x, a, r, perf_counter() - t0)


def dense_solve(S, lam, v):
    """Independent m-by-m LU oracle (tests/conftest.py:11-24, plain variant)."""
    A = np.asarray(S, dtype=np.float64)
    dense = A.T @ A + lam * np.eye(A.shape[1])
    return np.linalg.solve(dense, np.asarray(v, dtype=np.float64))


def rel_err(x, ref):
    """tests/conftest.py:27-29."""
    return float(np.linalg.norm(x - ref) / max(1.0, np.linalg.norm(ref)))


def phase_times(S: np.ndarray, v: np.ndarray, lam: float) -> dict:
    """Per-phase wall times of the reference path (SURVEY §6 breakdown), seconds."""
    A = np.ascontiguousarray(S, dtype=np.float64)
    out = {}
    t = perf_counter(); W = gram(A, lam); out["gram"] = perf_counter() - t
    t = perf_counter(); L = cholesky_lower(W); out["potrf"] = perf_counter() - t
    t = perf_counter(); t1 = A @ v; out["gemv_sv"] = perf_counter() - t
    t = perf_counter()
    t3 = solve_triangular(L, solve_triangular(L, t1, lower=True, check_finite=False),
                          lower=True, trans="T", check_finite=False)
    out["trsv"] = perf_counter() - t
    t = perf_counter(); x = (v - t3 @ A) / lam; out["gemv_stz"] = perf_counter() - t
    t = perf_counter(); residual(A, lam, v, x); out["residual"] = perf_counter() - t
    return out
