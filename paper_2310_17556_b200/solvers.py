"""Solver entry points of the damped Fisher system on B200 (mirror of fisher_solve.solvers).

``solve_chol`` is the hot path (solvers.py:151-206 of the reference): one call into
``fs_chol_solve`` of libfisher_b200.so runs Gram (tcgen05 SYRK) -> potrf -> TRSV pair
-> fused (v - S^T z)/lam epilogue -> fp64 residual diagnostics -> optional one-step
refinement, ordered on the current CUDA stream with a single host synchronisation.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass
from time import perf_counter

import numpy as np
import torch

from . import _lib
from .core import (
    EPS,
    DampedSystem,
    FactorizationError,
    Method,
    ScoreMatrix,
    Solution,
    Variant,
    WorkspaceMeter,
    PRECISIONS,
    _check,
    _dt,
    _stream,
    embed_complex,
    resolve_precision,
    stack_complex_vector,
)

DEFAULT_NAIVE_CAP = 4096            # solvers.py:38
DEFAULT_SIGMA_FLOOR = 1e-12         # solvers.py:39
REFINE_ABOVE_REL = 1e-10            # solvers.py:43 (_REFINE_ABOVE_REL)


def fp32_residual_bound(sigma2_max_over_lam: float) -> float:
    """Stated tolerance of the fp32 (tf32x3) mode: 4 u32 sigma_max^2 / lam."""
    return 4.0 * 2.0 ** -24 * sigma2_max_over_lam


@dataclass(frozen=True)
class CholWorkspace:
    """Lower Cholesky factor of the damped Gram matrix (solvers.py:57-71), device resident."""

    L: torch.Tensor   # n x n float64 CUDA tensor, upper triangle exactly zero

    @property
    def n(self) -> int:
        return int(self.L.shape[0])

    def solve_gram(self, b) -> np.ndarray:
        """Solve (L L^T) y = b by forward then back substitution on the GPU."""
        bt = torch.as_tensor(np.asarray(b, dtype=np.float64) if not isinstance(b, torch.Tensor) else b,
                             dtype=torch.float64).to(self.L.device).clone()
        ctx = _lib.context_for(self.L.device.index, self.n, 1)
        rc = ctx.lib.fs_trsv_pair(ctx.handle, self.L.data_ptr(), self.n, self.L.stride(0), bt.data_ptr(),
                                  _stream(self.L.device))
        _check(ctx, rc, "fs_trsv_pair")
        return bt.cpu().numpy() if not isinstance(b, torch.Tensor) else bt


def cholesky_lower_device(W: torch.Tensor) -> torch.Tensor:
    """In-place-safe lower Cholesky on the GPU with the reference's pivot contract (solvers.py:74-90)."""
    n = int(W.shape[0])
    L = W.to(torch.float64).contiguous().clone()
    L = torch.tril(L)  # the kernel reads the lower triangle and keeps the upper exactly zero
    ctx = _lib.context_for(L.device.index, n, 1)
    piv = ctypes.c_int64(-1)
    rc = ctx.lib.fs_potrf(ctx.handle, L.data_ptr(), n, L.stride(0), ctypes.byref(piv), _stream(L.device))
    if rc == _lib.FS_NOT_PD:
        raise FactorizationError(
            f"Gram matrix is not positive definite at pivot {piv.value}; retry with a larger damping",
            pivot=int(piv.value))
    _check(ctx, rc, "fs_potrf")
    return L


def _cholesky_lower(W) -> np.ndarray:
    """Host-array convenience mirror of solvers.py:74-90 (runs on the GPU)."""
    from .core import default_device
    Wt = torch.as_tensor(np.asarray(W, dtype=np.float64)).to(default_device())
    return cholesky_lower_device(Wt).cpu().numpy()


class _PinnedOut:
    """Page-locked fp64 output vectors for host solves, recycled once the caller has dropped the
    numpy array handed out (a D2H into pageable, freshly faulted memory costs ~2 ms per 8 MB on
    the GPU boxes; into pinned memory ~0.2 ms)."""

    def __init__(self, cap: int = 4):
        self.cap = cap
        self.pool: dict[int, list] = {}     # m -> [[pinned tensor, weakref to the array handed out]]

    def get(self, m: int) -> np.ndarray:
        slots = self.pool.setdefault(m, [])
        for slot in slots:
            if slot[1] is None or slot[1]() is None:
                arr = slot[0].numpy()
                slot[1] = weakref.ref(arr)
                return arr
        if len(slots) >= self.cap:
            return np.empty(m, dtype=np.float64)
        # allocate two at a time: a caller that keeps the previous result while solving again
        # (x = solve(...) in a loop) alternates between them without a cudaHostAlloc per call
        for _ in range(2 if not slots else 1):
            slots.append([torch.empty(m, dtype=torch.float64, pin_memory=True), None])
        slot = slots[-1]
        arr = slot[0].numpy()
        slot[1] = weakref.ref(arr)
        return arr


_pinned_out = _PinnedOut()


def _meter_slots(n: int, m: int, dtype: int, precision: int) -> int:
    lib = _lib.load()
    return int(lib.fs_workspace_bytes(n, m, dtype, precision)) // 8


def solve_chol(system: DampedSystem, meter: WorkspaceMeter | None = None, *, precision: str = "auto",
               refine: str | bool | int = "auto", diagnostics: bool = True) -> Solution:
    """Solve (S^T S + lam I) x = v through the n-by-n Gram factorization (solvers.py:197-206).

    precision: "fp64" (exact fp64 products, the reference's arithmetic), "f16x2" (default for
    fp32 scores: row-scaled two-plane fp16 split on the tensor cores), "tf32x3", or "auto".
    refine: "auto" applies the reference's one-step refinement rule (rel_residual > 1e-10,
    solvers.py:171-194) in fp64 mode and none in the fp32 modes, whose stated bound is
    4 u32 sigma_max^2/lam; True forces the reference rule; an int k > 1 runs up to k correction
    steps with the same factor and fp64 residuals (mixed-precision iterative refinement,
    SURVEY §8f-1), stopping at rel_residual <= 1e-10 or when a step no longer halves it —
    it contracts when u32 sigma_max^2/lam << 1; False disables refinement.
    diagnostics: compute abs/rel residual on the GPU (two extra passes over S), as the
    reference does inside solve_chol (solvers.py:160-170).
    """
    if system.S.is_complex:
        raise ValueError("solve_chol handles real scores; use solve_chol_hermitian")
    t0 = perf_counter()
    n, m = system.n, system.m
    prec = resolve_precision(precision, system.S.dtype)
    steps = 0
    if refine == "auto":
        steps = 1 if prec == "fp64" else 0
    elif isinstance(refine, bool):
        steps = 1 if refine else 0
    elif isinstance(refine, (int, np.integer)) and 0 <= int(refine) <= 255:
        steps = int(refine)
    else:
        raise ValueError(f"refine must be 'auto', a bool or a step count in [0, 255], got {refine!r}")
    do_refine = steps > 0
    if do_refine and not diagnostics:
        raise ValueError("refinement needs the residual diagnostics")
    flags = (_lib.FS_FLAG_RESIDUAL if diagnostics else 0) | ((_lib.FS_FLAG_REFINE | (steps << 8)) if do_refine else 0)
    dt = _lib.FS_F32 if system.S.dtype == torch.float32 else _lib.FS_F64
    device = system.S.device
    ctx = _lib.context_for(device.index, n, m)
    slots = _meter_slots(n, m, dt, PRECISIONS[prec])
    if meter is not None:
        meter.alloc(slots + m)
    piv = ctypes.c_int64(-1)
    res = (ctypes.c_double * 2)(float("nan"), float("nan"))
    Sh, vh = system.S.host_array, system.host_v
    if Sh is not None and vh is not None:
        # host system: one call streams S in row chunks overlapped with the Gram, returns x on the host
        x = _pinned_out.get(m)
        rc = ctx.lib.fs_chol_solve_host(ctx.handle, dt, PRECISIONS[prec], Sh.ctypes.data, n, m,
                                        Sh.strides[0] // Sh.itemsize, vh.ctypes.data, system.lam, x.ctypes.data,
                                        _lib.ALLREDUCE_FN(), None, flags, REFINE_ABOVE_REL, ctypes.byref(piv), res,
                                        _stream(device))
        what = "fs_chol_solve_host"
    else:
        S = system.S.tensor
        v = system.v_tensor
        x = torch.empty(m, dtype=torch.float64, device=S.device)
        rc = ctx.lib.fs_chol_solve(ctx.handle, dt, PRECISIONS[prec], S.data_ptr(), n, m, S.stride(0),
                                   v.data_ptr(), system.lam, x.data_ptr(), _lib.ALLREDUCE_FN(), None, flags,
                                   REFINE_ABOVE_REL, ctypes.byref(piv), res, _stream(S.device))
        what = "fs_chol_solve"
    if meter is not None:
        meter.free(slots)
    if rc == _lib.FS_NOT_PD:
        raise FactorizationError(
            f"Gram matrix is not positive definite at pivot {piv.value}; retry with a larger damping",
            pivot=int(piv.value))
    _check(ctx, rc, what)
    xo = x.cpu().numpy() if (system.S.host_origin and isinstance(x, torch.Tensor)) else x
    return Solution(x=xo, method=Method.CHOL, abs_residual=float(res[0]), rel_residual=float(res[1]),
                    wall_seconds=perf_counter() - t0, precision=prec)


def solve_chol_hermitian(system: DampedSystem, meter: WorkspaceMeter | None = None, *, precision: str = "auto",
                         refine: str | bool | int = "auto") -> Solution:
    """(S^H S + lam I) x = v for complex scores (solvers.py:209-213), through the real
    representation rho(S) = [[Re S, -Im S], [Im S, Re S]] (rho(S)^T rho(S) = rho(S^H S)): the plain
    route on 2n rows and 2m columns solves for [Re x; Im x] (fs_embed_complex + fs_chol_solve)."""
    if not system.S.is_complex:
        raise ValueError("solve_chol_hermitian expects complex scores; use solve_chol")
    t0 = perf_counter()
    m = system.m
    emb = embed_complex(system.S, 1)
    vhat = stack_complex_vector(system.v_tensor, system.S.real_dtype)
    inner = solve_chol(DampedSystem(emb, system.lam, vhat), meter, precision=precision, refine=refine)
    xh = inner.x
    x = torch.complex(xh[:m], xh[m:])
    xo = x.cpu().numpy() if system.S.host_origin else x
    return Solution(x=xo, method=Method.CHOL, abs_residual=inner.abs_residual, rel_residual=inner.rel_residual,
                    wall_seconds=perf_counter() - t0, precision=inner.precision)


def solve_realpart(system: DampedSystem, meter: WorkspaceMeter | None = None, *, precision: str = "auto",
                   refine: str | bool | int = "auto") -> Solution:
    """(Re[S^H S] + lam I) x = v for complex scores and a real v (solvers.py:216-240): the plain
    route on C = [Re S; Im S] (sr.py:61-70, built on the device by fs_embed_complex); the
    residual of the real-part operator equals C's plain residual."""
    if not system.S.is_complex:
        raise ValueError("real-part variant expects complex scores")
    if system.v_tensor.is_complex():
        raise ValueError("real-part variant requires a real right-hand side")
    t0 = perf_counter()
    C = embed_complex(system.S, 0)
    inner = solve_chol(DampedSystem(C, system.lam, system.v_tensor), meter, precision=precision, refine=refine)
    xo = inner.x.cpu().numpy() if system.S.host_origin else inner.x
    return Solution(x=xo, method=Method.CHOL, abs_residual=inner.abs_residual, rel_residual=inner.rel_residual,
                    wall_seconds=perf_counter() - t0, precision=inner.precision)


@dataclass(frozen=True)
class ThinSvd:
    """Thin SVD factors S = U diag(sigma) V^T (solvers.py ThinSvd): U n x r, sigma (r,), V m x r."""

    U: object
    sigma: object
    V: object

    @property
    def r(self) -> int:
        return int(self.sigma.shape[0])

    @property
    def m(self) -> int:
        return int(self.V.shape[0])


def _check_floor(sigma_floor) -> float:
    sigma_floor = float(sigma_floor)
    if not np.isfinite(sigma_floor) or sigma_floor < 0.0:
        raise ValueError(f"sigma_floor must be finite and >= 0, got {sigma_floor}")
    return sigma_floor


def eigh_gram(S: ScoreMatrix, precision: str = "auto") -> tuple[torch.Tensor, torch.Tensor, int]:
    """Eigenpairs of the Gram S S^T on the GPU (solvers.py:257-266): w descending (fp64, device),
    U (n x n fp64, device, column j <-> w[j]), and the Jacobi sweep count."""
    t = S.tensor
    n = S.n
    Gp = _gram_packed_unshifted(S, precision)
    ctx = _lib.context_for(t.device.index, n, S.m)
    w = torch.empty(n, dtype=torch.float64, device=t.device)
    U = torch.empty((n, n), dtype=torch.float64, device=t.device)
    sweeps = ctypes.c_int(0)
    rc = ctx.lib.fs_syevj_packed(ctx.handle, Gp.data_ptr(), n, w.data_ptr(), U.data_ptr(), n, ctypes.byref(sweeps),
                                 _stream(t.device))
    if rc == _lib.FS_ENOCONV:
        raise FactorizationError(f"eigendecomposition did not converge: {ctx.last_error()}")
    _check(ctx, rc, "fs_syevj_packed")
    return w, U, int(sweeps.value)


def _gram_packed_unshifted(S: ScoreMatrix, precision: str) -> torch.Tensor:
    t = S.tensor
    n, m = S.n, S.m
    prec = resolve_precision(precision, t.dtype)
    ctx = _lib.context_for(t.device.index, n, m)
    out = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device=t.device)
    rc = ctx.lib.fs_gram_packed(ctx.handle, _dt(t), PRECISIONS[prec], t.data_ptr(), n, m, t.stride(0), 0.0,
                                out.data_ptr(), _stream(t.device))
    _check(ctx, rc, "fs_gram_packed")
    return out


def thin_svd_eigh(S: ScoreMatrix, sigma_floor: float = DEFAULT_SIGMA_FLOOR, *, precision: str = "auto") -> ThinSvd:
    """Thin SVD via the eigendecomposition of the n-by-n Gram matrix (solvers.py:243-277) on the GPU.

    Eigenvalues made negative by round-off are clamped to zero; singular values at or below
    sigma_floor * sigma_max are truncated; V = S^T (U / sigma).  The Gram and the Jacobi
    eigensolver are this package's kernels; the explicit m x r factor V is one plain dense
    product (torch.matmul) — the solve route (solve_svd_eigh) never forms it.
    """
    sigma_floor = _check_floor(sigma_floor)
    if S.n > S.m:
        raise ValueError(f"thin_svd_eigh requires n <= m, got shape {S.shape}")
    w, U, _ = eigh_gram(S, precision)
    sigma = torch.sqrt(torch.clamp(w, min=0.0))
    keep = sigma > sigma_floor * sigma[0]
    U = U[:, keep].contiguous()
    sigma = sigma[keep].contiguous()
    if sigma.numel() == 0:
        V = torch.zeros((S.m, 0), dtype=torch.float64, device=U.device)
    else:
        V = S.tensor.to(torch.float64).T @ (U / sigma)
    if S.host_origin:
        return ThinSvd(U=U.cpu().numpy(), sigma=sigma.cpu().numpy(), V=V.cpu().numpy())
    return ThinSvd(U=U, sigma=sigma, V=V)


def solve_svd_eigh(system: DampedSystem, sigma_floor: float = DEFAULT_SIGMA_FLOOR, *, precision: str = "auto",
                   diagnostics: bool = True) -> Solution:
    """solve_svd_eigh (solvers.py:347-354): thin SVD through the Gram eigendecomposition, then
    x = V (sigma^2 + lam)^-1 V^T v + (v - V V^T v) / lam (solvers.py:315-317), residual against S.

    On the GPU (fs_eigh_solve): Gram + u = S v (same kernels and precision modes as solve_chol),
    Jacobi eigendecomposition, and the solve through S^T without forming V:
    x = (v - S^T z) / lam with z = U_r diag(1 / (w_r + lam)) U_r^T u over the kept eigenpairs.
    """
    sigma_floor = _check_floor(sigma_floor)
    t0 = perf_counter()
    S = system.S.tensor
    v = system.v_tensor
    n, m = system.n, system.m
    if n > m:
        raise ValueError(f"thin_svd_eigh requires n <= m, got shape {(n, m)}")
    prec = resolve_precision(precision, S.dtype)
    ctx = _lib.context_for(S.device.index, n, m)
    x = torch.empty(m, dtype=torch.float64, device=S.device)
    rank = ctypes.c_int64(0)
    res = (ctypes.c_double * 2)(float("nan"), float("nan"))
    flags = _lib.FS_FLAG_RESIDUAL if diagnostics else 0
    rc = ctx.lib.fs_eigh_solve(ctx.handle, _dt(S), PRECISIONS[prec], S.data_ptr(), n, m, S.stride(0), v.data_ptr(),
                               system.lam, sigma_floor, x.data_ptr(), _lib.ALLREDUCE_FN(), None, flags,
                               ctypes.byref(rank), res, _stream(S.device))
    if rc == _lib.FS_ENOCONV:
        raise FactorizationError(f"eigendecomposition did not converge: {ctx.last_error()}")
    _check(ctx, rc, "fs_eigh_solve")
    xo = x.cpu().numpy() if system.S.host_origin else x
    return Solution(x=xo, method=Method.SVD_EIGH, abs_residual=float(res[0]), rel_residual=float(res[1]),
                    wall_seconds=perf_counter() - t0, precision=prec)


def solve_svd_direct(system: DampedSystem, *, precision: str = "auto", diagnostics: bool = True) -> Solution:
    """solve_svd_direct (solvers.py:357-364, the "svda" comparison route): thin SVD of S, exact-zero
    singular values dropped (solvers.py:280-291), then the factor solve with the residual against S.

    The reference calls dgesdd; the paper's GPU svda called cuSOLVER gesvda, a Gram-based
    approximate tall-skinny SVD.  This route follows the paper's algorithm class: the thin SVD
    comes from the Jacobi eigendecomposition of S S^T (fs_eigh_solve) with NO floor — only
    singular values that are exactly zero (eigenvalues <= 0) are dropped, as in the reference.
    """
    sol = solve_svd_eigh(system, 0.0, precision=precision, diagnostics=diagnostics)
    return Solution(x=sol.x, method=Method.SVD_DIRECT, abs_residual=sol.abs_residual,
                    rel_residual=sol.rel_residual, wall_seconds=sol.wall_seconds, precision=sol.precision)
