"""Solver entry points of the damped Fisher system on B200 (mirror of fisher_solve.solvers).

``solve_chol`` is the hot path (solvers.py:151-206 of the reference): one call into
``fs_chol_solve`` of libfisher_b200.so runs Gram (tcgen05 SYRK) -> potrf -> TRSV pair
-> fused (v - S^T z)/lam epilogue -> fp64 residual diagnostics -> optional one-step
refinement, ordered on the current CUDA stream with a single host synchronisation.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass, replace
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
    as_scores,
    as_system,
    _check,
    _dt,
    _stream,
    embed_complex,
    gram_packed,
    hint_scales,
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
    """Lower Cholesky factor of the damped Gram matrix (solvers.py:57-71).  L is an n x n float64
    CUDA tensor (upper triangle exactly zero) or, as the reference holds it, a numpy array — then
    it is uploaded once for the solves."""

    L: object

    @property
    def n(self) -> int:
        return int(self.L.shape[0])

    def _device_L(self) -> torch.Tensor:
        if isinstance(self.L, torch.Tensor) and self.L.is_cuda:
            return self.L
        cached = self.__dict__.get("_dL")
        if cached is None:
            from .core import default_device
            cached = torch.as_tensor(np.ascontiguousarray(np.asarray(self.L, dtype=np.float64))).to(default_device())
            object.__setattr__(self, "_dL", cached)
        return cached

    def solve_gram(self, b) -> np.ndarray:
        """Solve (L L^T) y = b by forward then back substitution on the GPU."""
        L = self._device_L()
        bt = torch.as_tensor(np.asarray(b, dtype=np.float64) if not isinstance(b, torch.Tensor) else b,
                             dtype=torch.float64).to(L.device).clone()
        ctx = _lib.context_for(L.device.index, self.n, 1)
        rc = ctx.lib.fs_trsv_pair(ctx.handle, L.data_ptr(), self.n, L.stride(0), bt.data_ptr(), _stream(L.device))
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


AUTO_REFINE_STEPS = 4               # fp32 modes: z-space correction steps the "auto" rule may take
RESULT_PROMISE_REL = 1e-8           # solvers.py:41-42: the factored route promises rel_residual <= 1e-8


def _refine_steps(refine, prec: str) -> int:
    if isinstance(refine, str):
        if refine != "auto":
            raise ValueError(f"refine must be 'auto', a bool or a step count in [0, 255], got {refine!r}")
        # the reference rule (solvers.py:171-194): refine while rel_residual > 1e-10.  fp64 needs
        # one step at most (the reference's single correction pass); the fp32-split factors
        # refine z on the n x n system (contraction ~2^-21 kappa(W) per step, FS_FLAG_REFINE_Z)
        return 1 if prec == "fp64" else AUTO_REFINE_STEPS
    if isinstance(refine, bool):
        return 1 if refine else 0
    if isinstance(refine, (int, np.integer)) and 0 <= int(refine) <= 255:
        return int(refine)
    raise ValueError(f"refine must be 'auto', a bool or a step count in [0, 255], got {refine!r}")


def refine_flags(prec: str, steps: int) -> int:
    """fs_chol_solve refinement flags: fp64 -> the reference's x-space correction (solvers.py:183-194);
    the fp32-split modes -> z-space refinement on the n x n system (FS_FLAG_REFINE_Z)."""
    if steps <= 0:
        return 0
    return (_lib.FS_FLAG_REFINE if prec == "fp64" else _lib.FS_FLAG_REFINE_Z) | (min(int(steps), 255) << 8)


def _host_x(x: torch.Tensor) -> np.ndarray:
    """x (device fp64) -> a numpy array in page-locked memory (fast D2H; see _PinnedOut)."""
    out = _pinned_out.get(int(x.shape[0]))
    torch.from_numpy(out).copy_(x)
    return out


def solve_chol(system: DampedSystem, meter: WorkspaceMeter | None = None, *, precision: str = "auto",
               refine: str | bool | int = "auto", diagnostics: bool = True) -> Solution:
    """Solve (S^T S + lam I) x = v through the n-by-n Gram factorization (solvers.py:197-206).

    precision: "fp64" (exact fp64 products, the reference's arithmetic), "f16x2" (row-scaled
    two-plane fp16 split on the tensor cores), "tf32x3", or "auto" (fp64 scores -> fp64,
    float32 scores -> f16x2 with the result-quality guarantee below).
    refine: "auto" applies the reference's result rule (solvers.py:171-194): in fp64 mode its
    single x-space correction when rel_residual > 1e-10; in the fp32-split modes up to
    AUTO_REFINE_STEPS z-space steps (mixed-precision refinement of z = W^-1 S v on the n x n
    system with the split factor and exact fp64 residuals read off the fused x + y pass, one pass
    over S per step; it converges whatever sigma_max^2/lam is, because the n x n system is as
    well conditioned as W).  With precision="auto" as well, a float32 solve whose rel_residual
    still exceeds the reference's promise of 1e-8 (solvers.py:41-42) is recomputed in fp64 mode,
    so the drop-in default always meets the reference's result contract.  True = one step; an
    int k = up to k steps; False/0 = none (the raw fp32 mode, tolerance 4 u32 sigma_max^2/lam,
    SURVEY §8d).
    diagnostics: compute abs/rel residual on the GPU (two extra passes over S), as the
    reference does inside solve_chol (solvers.py:160-170).
    """
    system = as_system(system)
    if system.S.is_complex:
        raise ValueError("solve_chol handles real scores; use solve_chol_hermitian")
    t0 = perf_counter()
    n, m = system.n, system.m
    prec = resolve_precision(precision, system.S.dtype)
    steps = _refine_steps(refine, prec)
    do_refine = steps > 0
    if do_refine and not diagnostics:
        if refine == "auto":
            steps, do_refine = 0, False
        else:
            raise ValueError("refinement needs the residual diagnostics")
    flags = (_lib.FS_FLAG_RESIDUAL if diagnostics else 0) | (refine_flags(prec, steps) if do_refine else 0)
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
        # deferred host system: one call streams S in column chunks overlapped with the Gram and
        # returns x on the host
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
        hint_scales(ctx, system.S)
        rc = ctx.lib.fs_chol_solve(ctx.handle, dt, PRECISIONS[prec], S.data_ptr(), n, m, S.stride(0),
                                   v.data_ptr(), system.lam, x.data_ptr(), _lib.ALLREDUCE_FN(), None, flags,
                                   REFINE_ABOVE_REL, ctypes.byref(piv), res, _stream(S.device))
        what = "fs_chol_solve"
    if meter is not None:
        meter.free(slots)
    if rc == _lib.FS_NOT_PD:
        if precision == "auto" and prec != "fp64":
            # the split Gram carries ~2^-22 ||G|| of error, so W~ can lose definiteness where the
            # reference's fp64 W keeps it (near-dependent rows, lam below that error): decide in the
            # reference's arithmetic — its success, or its failure with its own pivot
            sol = solve_chol(system, meter, precision="fp64", refine=refine, diagnostics=diagnostics)
            return replace(sol, wall_seconds=perf_counter() - t0)
        raise FactorizationError(
            f"Gram matrix is not positive definite at pivot {piv.value}; retry with a larger damping",
            pivot=int(piv.value))
    _check(ctx, rc, what)
    if (precision == "auto" and refine == "auto" and prec != "fp64" and diagnostics
            and not float(res[1]) <= RESULT_PROMISE_REL):
        # the fp32-split factor could not reach the reference's promise: exact fp64 products
        sol = solve_chol(system, meter, precision="fp64", refine="auto", diagnostics=True)
        return replace(sol, wall_seconds=perf_counter() - t0)
    xo = _host_x(x) if (system.S.host_origin and isinstance(x, torch.Tensor)) else x
    return Solution(x=xo, method=Method.CHOL, abs_residual=float(res[0]), rel_residual=float(res[1]),
                    wall_seconds=perf_counter() - t0, precision=prec)


def solve_chol_hermitian(system: DampedSystem, meter: WorkspaceMeter | None = None, *, precision: str = "auto",
                         refine: str | bool | int = "auto") -> Solution:
    """(S^H S + lam I) x = v for complex scores (solvers.py:209-213), through the real
    representation rho(S) = [[Re S, -Im S], [Im S, Re S]] (rho(S)^T rho(S) = rho(S^H S)): the plain
    route on 2n rows and 2m columns solves for [Re x; Im x] (fs_embed_complex + fs_chol_solve)."""
    system = as_system(system)
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
    system = as_system(system)
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


def _shape_of(a) -> tuple:
    return tuple(a.shape)


@dataclass(frozen=True)
class ThinSvd:
    """Thin SVD factors S = U diag(sigma) V^H (core.py:226-267): U n x r and V m x r with
    orthonormal columns, sigma strictly positive and nonincreasing; r = 0 means numerically zero.
    The factors are numpy arrays for host-origin scores, CUDA tensors for device scores."""

    U: object
    sigma: object
    V: object

    def __post_init__(self):                 # core.py:237-253
        U, sigma, V = self.U, self.sigma, self.V
        if len(_shape_of(U)) != 2 or len(_shape_of(V)) != 2 or len(_shape_of(sigma)) != 1:
            raise ValueError("thin SVD factors have wrong ranks")
        r = _shape_of(sigma)[0]
        if _shape_of(U)[1] != r or _shape_of(V)[1] != r:
            raise ValueError(f"inconsistent retained rank: U has {_shape_of(U)[1]} columns, "
                             f"V has {_shape_of(V)[1]}, sigma has {r}")
        if r > min(_shape_of(U)[0], _shape_of(V)[0]):
            raise ValueError("retained rank exceeds min(n, m)")
        if r > 0:
            sg = sigma.detach().cpu().numpy() if isinstance(sigma, torch.Tensor) else np.asarray(sigma)
            if not np.all(sg > 0.0):
                raise ValueError("singular values must be strictly positive")
            if np.any(np.diff(sg) > 0.0):
                raise ValueError("singular values must be nonincreasing")

    @property
    def r(self) -> int:
        return int(_shape_of(self.sigma)[0])

    @property
    def n(self) -> int:
        return int(_shape_of(self.U)[0])

    @property
    def m(self) -> int:
        return int(_shape_of(self.V)[0])


def _check_floor(sigma_floor) -> float:
    sigma_floor = float(sigma_floor)
    if not np.isfinite(sigma_floor) or sigma_floor < 0.0:
        raise ValueError(f"sigma_floor must be finite and >= 0, got {sigma_floor}")
    return sigma_floor


def eigh_gram(S: ScoreMatrix, precision: str = "auto") -> tuple[torch.Tensor, torch.Tensor, int]:
    """Eigenpairs of the Gram S S^T on the GPU (solvers.py:257-266): w descending (fp64, device),
    U (n x n fp64, device, column j <-> w[j]), and the Jacobi sweep count (real scores)."""
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
    dt = _dt(t)
    prec = resolve_precision(precision, t.dtype)
    ctx = _lib.context_for(t.device.index, n, m)
    out = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device=t.device)
    hint_scales(ctx, S)
    rc = ctx.lib.fs_gram_packed(ctx.handle, dt, PRECISIONS[prec], t.data_ptr(), n, m, t.stride(0), 0.0,
                                out.data_ptr(), _stream(t.device))
    _check(ctx, rc, "fs_gram_packed")
    return out


def _apply_rows(T: torch.Tensor, X: torch.Tensor, lower: bool = False) -> torch.Tensor:
    """Y = T X on the device (fs_apply_rows, fp64 tensor cores): T r x n fp64, X n x m (a real
    score-layout matrix, fp32 or fp64, unit column stride) -> Y r x m fp64, 16-byte aligned rows.
    lower: T is lower triangular (fs_apply_rows_lower skips its zero upper part)."""
    r, n = int(T.shape[0]), int(T.shape[1])
    m = int(X.shape[1])
    T = T.to(torch.float64).contiguous()
    ldy = -(-m // 2) * 2
    Y = torch.empty((r, ldy), dtype=torch.float64, device=X.device)[:, :m]
    ctx = _lib.context_for(X.device.index, n, m)
    ldT = T.stride(0) if r > 1 else n          # a 1-row tensor may carry any row stride
    fn = ctx.lib.fs_apply_rows_lower if lower else ctx.lib.fs_apply_rows
    rc = fn(ctx.handle, _dt(X), T.data_ptr(), r, n, ldT, X.data_ptr(), m, X.stride(0), Y.data_ptr(), Y.stride(0),
            _stream(X.device))
    _check(ctx, rc, "fs_apply_rows")
    return Y


def thin_svd_eigh(S: ScoreMatrix, sigma_floor: float = DEFAULT_SIGMA_FLOOR, *, precision: str = "auto") -> ThinSvd:
    """Thin SVD via the eigendecomposition of the n-by-n Gram matrix (solvers.py:243-277) on the GPU.

    Eigenvalues made negative by round-off are clamped to zero; singular values at or below
    sigma_floor * sigma_max are truncated; V = S^T (U / sigma), formed as V^T = (U / sigma)^T S by
    this package's fp64 tensor-core GEMM (fs_apply_rows).  Complex scores: the eigenpairs of
    S S^H come from the Hermitian Jacobi eigensolver (fs_heevj_packed) on the Gram of
    [Re S; Im S], and V^H = (U / sigma)^H S through the real representation.
    """
    sigma_floor = _check_floor(sigma_floor)
    S = as_scores(S)
    if S.n > S.m:
        raise ValueError(f"thin_svd_eigh requires n <= m, got shape {S.shape}")
    if S.is_complex:
        return _thin_svd_eigh_complex(S, sigma_floor, precision)
    w, U, _ = eigh_gram(S, precision)
    sigma = torch.sqrt(torch.clamp(w, min=0.0))
    keep = sigma > sigma_floor * sigma[0]
    U = U[:, keep].contiguous()
    sigma = sigma[keep].contiguous()
    if sigma.numel() == 0:
        V = torch.zeros((S.m, 0), dtype=torch.float64, device=U.device)
    else:
        V = _apply_rows((U / sigma).T, S.tensor).T      # V^T = (U / sigma)^T S  (r x m)
    if S.host_origin:
        return ThinSvd(U=U.cpu().numpy(), sigma=sigma.cpu().numpy(), V=np.ascontiguousarray(V.cpu().numpy()))
    return ThinSvd(U=U, sigma=sigma, V=V)


def _thin_svd_eigh_complex(S: ScoreMatrix, sigma_floor: float, precision: str) -> ThinSvd:
    """Complex scores (solvers.py:258-276 with S S^H and V = S^H U / sigma): the Gram of
    C = [Re S; Im S] (one real SYRK on 2n rows), the Hermitian eigenpairs from fs_heevj_packed,
    and V^H = (U / sigma)^H S as two real fs_apply_rows products on C:
    Re V^H = [Re B^T, Im B^T] C and Im V^H = [-Im B^T, Re B^T] C with B = U / sigma."""
    n, m = S.n, S.m
    C = embed_complex(S, 0)
    G2 = gram_packed(C, 0.0, precision)
    dev = G2.device
    ctx = _lib.context_for(dev.index, 2 * n, m)
    w = torch.empty(n, dtype=torch.float64, device=dev)
    Ui = torch.empty((n, n, 2), dtype=torch.float64, device=dev)
    sweeps = ctypes.c_int(0)
    rc = ctx.lib.fs_heevj_packed(ctx.handle, G2.data_ptr(), n, w.data_ptr(), Ui.data_ptr(), n, ctypes.byref(sweeps),
                                 _stream(dev))
    if rc == _lib.FS_ENOCONV:
        raise FactorizationError(f"eigendecomposition did not converge: {ctx.last_error()}")
    _check(ctx, rc, "fs_heevj_packed")
    U = torch.view_as_complex(Ui)
    sigma = torch.sqrt(torch.clamp(w, min=0.0))
    keep = sigma > sigma_floor * sigma[0]
    U = U[:, keep].contiguous()
    sigma = sigma[keep].contiguous()
    r = int(sigma.shape[0])
    if r == 0:
        V = torch.zeros((m, 0), dtype=torch.complex128, device=dev)
    else:
        B = U / sigma
        Bt_re, Bt_im = B.real.T, B.imag.T
        T = torch.cat([torch.cat([Bt_re, Bt_im], dim=1), torch.cat([-Bt_im, Bt_re], dim=1)], dim=0)   # 2r x 2n
        Y = _apply_rows(T, C.tensor)                         # [Re V^H; Im V^H]  (2r x m)
        V = torch.complex(Y[:r], -Y[r:]).T                   # V = (V^H)^H
    if S.host_origin:
        return ThinSvd(U=U.cpu().numpy(), sigma=sigma.cpu().numpy(), V=np.ascontiguousarray(V.cpu().numpy()))
    return ThinSvd(U=U, sigma=sigma, V=V)


def solve_svd_eigh(system: DampedSystem, sigma_floor: float = DEFAULT_SIGMA_FLOOR, *, precision: str = "auto",
                   diagnostics: bool = True, refine: str | bool | int = "auto") -> Solution:
    """solve_svd_eigh (solvers.py:347-354): thin SVD through the Gram eigendecomposition, then
    x = V (sigma^2 + lam)^-1 V^T v + (v - V V^T v) / lam (solvers.py:315-317), residual against S.

    On the GPU (fs_eigh_solve): Gram + u = S v (same kernels and precision modes as solve_chol),
    Jacobi eigendecomposition, and the solve through S^T without forming V:
    x = (v - S^T z) / lam with z = U_r diag(1 / (w_r + lam)) U_r^T u over the kept eigenpairs.
    Complex scores (S^H S + lam I, the HERMITIAN residual as solvers.py:319-320 picks): the same
    route on the real representation rho(S) = [[Re S, -Im S], [Im S, Re S]] for [Re x; Im x]
    (rho(S) rho(S)^T = rho(S S^H) has every eigenvalue of S S^H twice, so the floor keeps or drops
    both copies and the solve is the complex one).
    refine: the reference's eigh route has no correction step, so fp64 mode never refines; in the
    fp32-split modes "auto" (with diagnostics) takes up to AUTO_REFINE_STEPS z-space steps as in
    solve_chol, the correction solve being the same kept-eigenpair apply: z converges to the fp64
    route's z = U_r diag(1 / (w_r + lam)) U_r^T u, i.e. the float32 default reaches the result the
    reference computes in fp64.  An int k = up to k steps; False/0 = the raw fp32 route.
    """
    return _eigh_route(as_system(system), _check_floor(sigma_floor), precision, diagnostics, Method.SVD_EIGH,
                       refine)


def _eigh_route(system: DampedSystem, sigma_floor: float, precision: str, diagnostics: bool,
                method: Method, refine: str | bool | int = "auto") -> Solution:
    t0 = perf_counter()
    if system.n > system.m:
        raise ValueError(f"thin_svd_eigh requires n <= m, got shape {(system.n, system.m)}")
    if system.S.is_complex:
        m = system.m
        emb = embed_complex(system.S, 1)
        vhat = stack_complex_vector(system.v_tensor, system.S.real_dtype)
        inner = _eigh_route(DampedSystem(emb, system.lam, vhat), sigma_floor, precision, diagnostics, method,
                            refine)
        x = torch.complex(inner.x[:m], inner.x[m:])
        xo = x.cpu().numpy() if system.S.host_origin else x
        return replace(inner, x=xo, wall_seconds=perf_counter() - t0)
    S = system.S.tensor
    v = system.v_tensor
    n, m = system.n, system.m
    prec = resolve_precision(precision, S.dtype)
    ctx = _lib.context_for(S.device.index, n, m)
    x = torch.empty(m, dtype=torch.float64, device=S.device)
    rank = ctypes.c_int64(0)
    res = (ctypes.c_double * 2)(float("nan"), float("nan"))
    steps = _refine_steps(refine, prec)
    if prec == "fp64":
        steps = 0
    if steps > 0 and not diagnostics:
        if refine != "auto":
            raise ValueError("refinement needs the residual diagnostics")
        steps = 0
    flags = (_lib.FS_FLAG_RESIDUAL if diagnostics else 0) | (refine_flags(prec, steps) if steps > 0 else 0)
    hint_scales(ctx, system.S)
    rc = ctx.lib.fs_eigh_solve(ctx.handle, _dt(S), PRECISIONS[prec], S.data_ptr(), n, m, S.stride(0), v.data_ptr(),
                               system.lam, sigma_floor, x.data_ptr(), _lib.ALLREDUCE_FN(), None, flags,
                               ctypes.byref(rank), res, _stream(S.device))
    if rc == _lib.FS_ENOCONV:
        raise FactorizationError(f"eigendecomposition did not converge: {ctx.last_error()}")
    _check(ctx, rc, "fs_eigh_solve")
    xo = _host_x(x) if system.S.host_origin else x
    return Solution(x=xo, method=method, abs_residual=float(res[0]), rel_residual=float(res[1]),
                    wall_seconds=perf_counter() - t0, precision=prec)


def solve_svd_from_factors(svd: ThinSvd, lam: float, v, *, source: ScoreMatrix | None = None,
                           method: Method = Method.SVD_EIGH) -> Solution:
    """x = V (sigma^2 + lam)^-1 V^H v + (v - V V^H v) / lam from thin SVD factors (solvers.py:294-344),
    on the GPU: with V^H in the score layout (r x m), t = V^H v is fs_gemv_rows and
    x = (v - V z) / lam with z = t sigma^2 / (sigma^2 + lam) is fs_gemv_cols_solve (the chol
    route's x pass; the same algebra as the reference, never forming V V^H).  Rank 0 gives
    x = v / lam exactly.  Residuals: against ``source`` when given (HERMITIAN for complex
    scores), else against the operator V diag(sigma^2) V^H + lam I the factors span.  Complex
    factors run on the real representation of V^H (fs_embed_complex)."""
    from .core import _coerce_damping, _to_device_tensor, default_device
    t0 = perf_counter()
    lam = _coerce_damping(lam)
    if source is not None:
        source = as_scores(source)
    dev = svd.V.device if isinstance(svd.V, torch.Tensor) else (
        source.device if source is not None else default_device())
    vt = _to_device_tensor(v, "right-hand side", dev, force_copy=isinstance(v, torch.Tensor) and v.is_cuda)
    if vt.dim() != 1 or vt.shape[0] != svd.m:
        raise ValueError(f"right-hand side has shape {tuple(vt.shape)}, expected ({svd.m},)")
    host_out = not isinstance(svd.V, torch.Tensor)
    V = torch.as_tensor(svd.V, device=dev)
    sigma = torch.as_tensor(svd.sigma, device=dev, dtype=torch.float64)
    m, r = svd.m, svd.r
    cplx = V.is_complex() or vt.is_complex()
    if cplx:
        vhat = stack_complex_vector(vt.to(torch.complex128), torch.float64)
    else:
        vhat = vt.to(torch.float64).contiguous()
    if r == 0:
        xhat = vhat / lam
    else:
        if cplx:
            Vh = ScoreMatrix(V.to(torch.complex128).conj().T.contiguous())
            E = embed_complex(Vh, 1).tensor                 # rho(V^H): 2r x 2m
            d = torch.cat([sigma, sigma])
        else:
            E = _to_device_tensor(V.to(torch.float64).T, "right factor", dev)   # V^T: r x m, aligned
            d = sigma
        rows, cols = int(E.shape[0]), int(E.shape[1])
        ctx = _lib.context_for(dev.index, rows, cols)
        st = _stream(dev)
        t = torch.empty(rows, dtype=torch.float64, device=dev)
        rc = ctx.lib.fs_gemv_rows(ctx.handle, _dt(E), E.data_ptr(), rows, cols, E.stride(0), vhat.data_ptr(),
                                  _lib.FS_F64, t.data_ptr(), st)
        _check(ctx, rc, "fs_gemv_rows")
        z = t * (d * d) / (d * d + lam)
        xhat = torch.empty(cols, dtype=torch.float64, device=dev)
        rc = ctx.lib.fs_gemv_cols_solve(ctx.handle, _dt(E), E.data_ptr(), rows, cols, E.stride(0), z.data_ptr(),
                                        vhat.data_ptr(), _lib.FS_F64, lam, 0, xhat.data_ptr(), st)
        _check(ctx, rc, "fs_gemv_cols_solve")
    x = torch.complex(xhat[:m], xhat[m:]) if cplx else xhat
    if source is not None:
        from .core import residual as _residual
        system = DampedSystem(source, lam, vt)
        abs_res, rel_res = _residual(system, x, Variant.HERMITIAN if source.is_complex else Variant.PLAIN)
    elif r == 0:
        abs_res = float(torch.linalg.vector_norm(lam * xhat - vhat))
        rel_res = abs_res / max(float(torch.linalg.vector_norm(vhat)), EPS)
    else:
        y = torch.empty(rows, dtype=torch.float64, device=dev)
        rc = ctx.lib.fs_gemv_rows(ctx.handle, _dt(E), E.data_ptr(), rows, cols, E.stride(0), xhat.data_ptr(),
                                  _lib.FS_F64, y.data_ptr(), st)
        _check(ctx, rc, "fs_gemv_rows")
        y *= d * d
        sums = torch.empty(2, dtype=torch.float64, device=dev)
        rc = ctx.lib.fs_residual_cols(ctx.handle, _dt(E), E.data_ptr(), rows, cols, E.stride(0), y.data_ptr(),
                                      xhat.data_ptr(), vhat.data_ptr(), _lib.FS_F64, lam, None, sums.data_ptr(), st)
        _check(ctx, rc, "fs_residual_cols")
        rr, vv = sums.cpu().tolist()
        abs_res = float(np.sqrt(rr))
        rel_res = abs_res / max(float(np.sqrt(vv)), EPS)
    xo = x.cpu().numpy() if host_out or (source is not None and source.host_origin) else x
    return Solution(x=xo, method=method, abs_residual=abs_res, rel_residual=rel_res,
                    wall_seconds=perf_counter() - t0, precision="fp64")


def thin_svd_direct(S: ScoreMatrix) -> ThinSvd:
    """Thin SVD of S itself (solvers.py:280-291; the reference calls dgesdd): exact-zero singular
    values dropped.  GPU route: shifted CholeskyQR3 of S^H (fp64 tensor-core
    Gram, potrf, triangular inverse and fs_apply_rows), then a one-sided Jacobi SVD of the n x n
    triangular factor (fs_svd_direct).  Tall S (n > m) is handled through S^T."""
    return _svda(as_scores(S), want_factors=True)


def solve_svd_direct(system: DampedSystem, *, precision: str = "auto", diagnostics: bool = True) -> Solution:
    """solve_svd_direct (solvers.py:357-364, the "svda" comparison route): thin SVD of S (see
    thin_svd_direct), then the factor solve with the residual against S.  The solve never forms
    V: with S = U diag(sigma) V^T, x = (v - S^T z)/lam and z = U diag(1/(sigma^2 + lam)) U^T S v
    (the eigh route's algebra with w = sigma^2 from the SVD, not from the Gram)."""
    t0 = perf_counter()
    system = as_system(system)
    if system.S.is_complex:
        raise ValueError("solve_svd_direct: complex scores are not supported on the GPU svd route")
    sol = _svda(system.S, want_factors=False, system=system, diagnostics=diagnostics)
    return replace(sol, wall_seconds=perf_counter() - t0)


U64 = 2.0 ** -53


def _potrf_device(Gp: torch.Tensor, n: int, shift: float) -> torch.Tensor | None:
    """L = chol(unpack(Gp) + shift I) on the device, or None on breakdown."""
    dev = Gp.device
    ctx = _lib.context_for(dev.index, n, 1)
    W = torch.empty((n, n), dtype=torch.float64, device=dev)
    st = _stream(dev)
    rc = ctx.lib.fs_unpack_lower(ctx.handle, Gp.data_ptr(), n, float(shift), W.data_ptr(), n, st)
    _check(ctx, rc, "fs_unpack_lower")
    piv = ctypes.c_int64(-1)
    rc = ctx.lib.fs_potrf(ctx.handle, W.data_ptr(), n, n, ctypes.byref(piv), st)
    if rc == _lib.FS_NOT_PD:
        return None
    _check(ctx, rc, "fs_potrf")
    return W


def _tri_inverse(L: torch.Tensor) -> torch.Tensor:
    n = int(L.shape[0])
    ctx = _lib.context_for(L.device.index, n, 1)
    out = torch.empty((n, n), dtype=torch.float64, device=L.device)
    rc = ctx.lib.fs_tri_inverse(ctx.handle, L.data_ptr(), n, L.stride(0), out.data_ptr(), n, _stream(L.device))
    _check(ctx, rc, "fs_tri_inverse")
    return out


def _jacobi_svd(A: torch.Tensor):
    n = int(A.shape[0])
    dev = A.device
    ctx = _lib.context_for(dev.index, n, 1)
    sigma = torch.empty(n, dtype=torch.float64, device=dev)
    U = torch.empty((n, n), dtype=torch.float64, device=dev)
    Zt = torch.empty((n, n), dtype=torch.float64, device=dev)
    sweeps = ctypes.c_int(0)
    rc = ctx.lib.fs_jacobi_svd(ctx.handle, A.data_ptr(), n, A.stride(0), sigma.data_ptr(), U.data_ptr(), n,
                               Zt.data_ptr(), n, ctypes.byref(sweeps), _stream(dev))
    if rc == _lib.FS_ENOCONV:
        raise FactorizationError(f"SVD did not converge: {ctx.last_error()}")
    _check(ctx, rc, "fs_jacobi_svd")
    return sigma, U, Zt


def _svda(S: ScoreMatrix, want_factors: bool, system: DampedSystem | None = None, diagnostics: bool = True):
    """The direct-SVD route on the GPU (see thin_svd_direct).  Shifted CholeskyQR3 (Fukaya,
    Kannan, Nakatsukasa, Zhang, Yamamoto 2020) of the tall X = S^T: the first Gram is shifted by
    s = 11 (m n + n (n + 1)) u ||S||_F^2 so its Cholesky factor exists for cond(S) up to ~1/u, and
    two plain CholeskyQR steps restore Q's orthogonality to O(u); every Gram is the exact-product
    fp64 SYRK, every Q^T <- L^-1 Q^T and factor product is fs_apply_rows.  Then S = L Q^T and
    the one-sided Jacobi SVD of L (not of a Gram: no squared condition number) gives the
    singular triplets.  A later step whose Gram is singular (exact rank deficiency: a zero or
    repeated row) is shifted as well, and the directions that stay at the shift's noise level
    (sigma <= sqrt(n m) u sigma_max) are dropped as numerically zero — the reference's dgesdd
    keeps tiny nonzero values there, which differ from run to run of any algorithm."""
    if S.is_complex:
        raise ValueError("thin_svd_direct: complex scores are not supported on the GPU svd route")
    from .core import _to_device_tensor
    n, m = S.n, S.m
    if n > m:
        # tall S: the thin SVD of S^T (wide), factors swapped (S = U s V^T <=> S^T = V s U^T)
        X = _to_device_tensor(S.tensor.T, "score matrix", S.tensor.device, force_copy=True)
        ST = ScoreMatrix._owned(X, host_origin=S.host_origin)
        if want_factors:
            f = _svda(ST, True)
            return ThinSvd(U=f.V, sigma=f.sigma, V=f.U)
        sigma, U, Zt, Qt, r = _svda_core(ST)
        # S = (Q Z) diag(sigma) W^T: S's left factors are Q Z (n x r), formed as (Z^T Q^T)^T
        Uleft = _apply_rows(Zt[:r], Qt).T.contiguous() if r else torch.zeros((n, 0), dtype=torch.float64,
                                                                               device=X.device)
        return _factor_solve(system, Uleft, sigma[:r], diagnostics)
    Gp = gram_packed(S, 0.0, "fp64")
    fast = _svda_gram_route(Gp, n)
    if fast is not None:
        sigma, U = fast
        if not want_factors:
            return _factor_solve(system, U, sigma, diagnostics)
        Vt = _apply_rows((U.T / sigma[:, None]).contiguous(), S.tensor)   # V^T = diag(1/sigma) U^T S
        if S.host_origin:
            return ThinSvd(U=U.cpu().numpy(), sigma=sigma.cpu().numpy(), V=np.ascontiguousarray(Vt.T.cpu().numpy()))
        return ThinSvd(U=U, sigma=sigma, V=Vt.T)
    sigma, U, Zt, Qt, r = _svda_core(S, Gp)
    if not want_factors:
        return _factor_solve(system, U[:, :r].contiguous(), sigma[:r], diagnostics)
    dev = S.tensor.device
    if r == 0:
        Uo = torch.zeros((n, 0), dtype=torch.float64, device=dev)
        so = torch.zeros(0, dtype=torch.float64, device=dev)
        V = torch.zeros((m, 0), dtype=torch.float64, device=dev)
    else:
        Uo = U[:, :r].contiguous()
        so = sigma[:r].contiguous()
        V = _apply_rows(Zt[:r], Qt).T                    # V^T = Z^T Q^T
    if S.host_origin:
        return ThinSvd(U=Uo.cpu().numpy(), sigma=so.cpu().numpy(), V=np.ascontiguousarray(V.cpu().numpy()))
    return ThinSvd(U=Uo, sigma=so, V=V)


# The svd route's well-conditioned fast path: when the exact-product fp64 Gram G = S S^T certifies
# cond(S)^2 = w_max / w_min <= 1/SVDA_GRAM_RATIO (cond(S) <= 100), the thin SVD comes from G's eigendecomposition
# (sigma = sqrt(w), U = G's eigenvectors — the Gram-based algorithm class of the paper's cuSOLVER
# gesvda).  G's rounding error is a few u ||S||^2, so each sigma_i^2 carries a relative error of
# at most ~u w_max / w_i <= 1e4 u ~ 2e-12 (V's orthonormality likewise): well inside the 1e-8 that
# dgesdd's results are compared at.
# Anything worse conditioned (or rank deficient) takes the shifted CholeskyQR3 + one-sided Jacobi
# route, whose accuracy does not depend on cond(S).  FS_SVDA_GRAM=0 forces that route.
SVDA_GRAM_RATIO = 1e-4


def _syevj_device(Gp: torch.Tensor, n: int):
    """(w descending, U) of the packed symmetric Gram on the device (fs_syevj_packed)."""
    dev = Gp.device
    ctx = _lib.context_for(dev.index, n, 1)
    w = torch.empty(n, dtype=torch.float64, device=dev)
    U = torch.empty((n, n), dtype=torch.float64, device=dev)
    sweeps = ctypes.c_int(0)
    rc = ctx.lib.fs_syevj_packed(ctx.handle, Gp.data_ptr(), n, w.data_ptr(), U.data_ptr(), n, ctypes.byref(sweeps),
                                 _stream(dev))
    if rc == _lib.FS_ENOCONV:
        raise FactorizationError(f"eigendecomposition did not converge: {ctx.last_error()}")
    _check(ctx, rc, "fs_syevj_packed")
    return w, U


def _svda_gram_route(Gp: torch.Tensor, n: int):
    """(sigma, U) from the Gram when it certifies a well-conditioned S, else None."""
    import os
    if os.environ.get("FS_SVDA_GRAM", "1") == "0" or n > 16384:
        return None
    w, U = _syevj_device(Gp, n)
    wh = w.cpu().numpy()
    if not (wh[0] > 0.0 and wh[-1] >= SVDA_GRAM_RATIO * wh[0]):
        return None
    return torch.sqrt(w), U


def _svda_core(S: ScoreMatrix, Gp: torch.Tensor | None = None):
    """-> (sigma descending, W (n x n), Z^T (n x n), Q^T (n x m fp64), kept rank r) with S = L Q^T,
    L = W diag(sigma) Z^T.  Gp: S's fp64 Gram when the caller has it already."""
    X = S.tensor
    n, m = S.n, S.m
    dev = X.device
    if Gp is None:
        Gp = gram_packed(S, 0.0, "fp64")
    diag = torch.arange(n, device=dev, dtype=torch.int64)
    fro2 = float(Gp[diag * (diag + 1) // 2 + diag].sum())
    if fro2 == 0.0:          # exactly zero scores: every singular value is an exact zero (dropped)
        z = torch.zeros(0, dtype=torch.float64, device=dev)
        return z, torch.zeros((n, n), dtype=torch.float64, device=dev), torch.zeros((n, n), dtype=torch.float64,
                                                                                   device=dev), None, 0
    shift = 11.0 * (m * n + n * (n + 1)) * U64 * fro2
    L = _potrf_device(Gp, n, shift)
    if L is None:
        raise FactorizationError("SVD did not converge: the shifted CholeskyQR Gram is not positive definite")
    Lacc = L
    Qt = _apply_rows(_tri_inverse(L), X, lower=True)
    deficient = False
    for _ in range(2):
        Gq = gram_packed(ScoreMatrix._owned(Qt), 0.0, "fp64")
        Lk = _potrf_device(Gq, n, 0.0)
        if Lk is None:       # exact rank deficiency: shift this step too
            deficient = True
            q2 = float(Gq[diag * (diag + 1) // 2 + diag].sum())
            Lk = _potrf_device(Gq, n, 11.0 * (m * n + n * (n + 1)) * U64 * max(q2, 1.0))
            if Lk is None:
                raise FactorizationError("SVD did not converge: CholeskyQR breakdown")
        Lacc = _apply_rows(Lacc, Lk, lower=True)   # a product of lower triangular factors
        Qt = _apply_rows(_tri_inverse(Lk), Qt, lower=True)
    sigma, W, Zt = _jacobi_svd(Lacc)
    sg = sigma.cpu().numpy()
    cut = np.sqrt(float(n) * m) * U64 * sg[0] if deficient else 0.0
    r = int(np.count_nonzero(sg > cut))
    return sigma, W, Zt, Qt, r


def _factor_solve(system: DampedSystem, U: torch.Tensor, sigma: torch.Tensor, diagnostics: bool) -> Solution:
    """x = (v - S^T z)/lam, z = U diag(1/(sigma^2 + lam)) U^T S v (fs_factor_solve), residual against S."""
    t0 = perf_counter()
    S = system.S.tensor
    v = system.v_tensor
    n, m = system.n, system.m
    r = int(sigma.shape[0])
    ctx = _lib.context_for(S.device.index, n, m)
    x = torch.empty(m, dtype=torch.float64, device=S.device)
    w = (sigma * sigma).contiguous()
    Uc = U.contiguous() if r else torch.zeros((n, 1), dtype=torch.float64, device=S.device)
    res = (ctypes.c_double * 2)(float("nan"), float("nan"))
    flags = _lib.FS_FLAG_RESIDUAL if diagnostics else 0
    rc = ctx.lib.fs_factor_solve(ctx.handle, _dt(S), S.data_ptr(), n, m, S.stride(0), v.data_ptr(), system.lam,
                                 Uc.data_ptr(), max(r, 1), w.data_ptr() if r else None, r, x.data_ptr(), flags, res,
                                 _stream(S.device))
    _check(ctx, rc, "fs_factor_solve")
    xo = _host_x(x) if system.S.host_origin else x
    return Solution(x=xo, method=Method.SVD_DIRECT, abs_residual=float(res[0]), rel_residual=float(res[1]),
                    wall_seconds=perf_counter() - t0, precision="fp64")


def resolve_solver(system: DampedSystem, method, variant=Variant.PLAIN, f=None, tol=1e-10, max_iter=None,
                   naive_cap=DEFAULT_NAIVE_CAP):
    """Map (method, variant, scalar kind) to a zero-argument solve callable (bench.py:183-219).

    Raises ValueError on method/kind mismatches, as the reference does.  The GPU path provides
    chol (plain / hermitian / realpart), eigh and svd; the reference's CPU-only baselines
    (naive, cg, rvb) are out of this package's scope and raise ValueError naming them."""
    system = as_system(system)
    method = Method(getattr(method, "value", method))
    variant = Variant(getattr(variant, "value", variant))
    is_complex = system.S.is_complex
    if method is Method.CHOL:
        if variant is Variant.PLAIN:
            if is_complex:
                raise ValueError("plain chol needs real scores; pick hermitian or realpart")
            return lambda: solve_chol(system)
        if variant is Variant.HERMITIAN:
            if not is_complex:
                raise ValueError("hermitian variant needs complex scores")
            return lambda: solve_chol_hermitian(system)
        if not is_complex:
            raise ValueError("real-part variant needs complex scores")
        return lambda: solve_realpart(system)
    if method in (Method.NAIVE, Method.CG, Method.RVB):
        raise ValueError(f"method {method.value} is a CPU baseline of the reference; the B200 path provides "
                         "chol, eigh and svd")
    if variant is not Variant.PLAIN:
        raise ValueError(f"method {method.value} supports the plain variant only")
    if method is Method.SVD_EIGH:
        return lambda: solve_svd_eigh(system)
    if method is Method.SVD_DIRECT:
        return lambda: solve_svd_direct(system)
    raise ValueError(f"unknown method: {method!r}")
