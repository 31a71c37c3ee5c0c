"""Column-sharded multi-GPU Cholesky solve.

Rank k owns the contiguous column block S[:, m_k:m_{k+1}] and v[m_k:m_{k+1}] as its own
row-major n x m_k allocation.  Per solve:

    packed = [G_k lower-packed (n(n+1)/2) | u_k = S_k v_k (n)]   (rank-local, tcgen05 SYRK + GEMV)
    all_reduce(packed)                                              (the only O(n^2) exchange)
    L = chol(G + lam I); z = L^-T L^-1 u                            (redundant on every rank)
    x_k = (v_k - S_k^T z) / lam                                     (rank-local, no communication)

The residual diagnostics add two tiny all-reduces (y = S x: n doubles; the norm pair).
The host logic here is backend-agnostic: `CudaStageOps` binds the C ABI of
libfisher_b200.so on torch CUDA tensors (the product); the CPU tests drive the same
`sharded_solve_chol` with a numpy stage implementation over a gloo process group.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Callable, Protocol

import numpy as np
import torch

from . import _lib
from .core import EPS, FactorizationError, _check, _dt, _stream, resolve_precision, PRECISIONS
from .solvers import REFINE_ABOVE_REL, refine_flags


def column_shard(m: int, world: int, rank: int) -> tuple[int, int]:
    """[m_k, m_{k+1}) with m_k = floor(k m / P): contiguous, sizes differ by at most one."""
    return (rank * m) // world, ((rank + 1) * m) // world


class StageOps(Protocol):
    def gram_partial(self, S, out) -> None: ...          # out[:T] = lower-packed S S^T (no shift)
    def gemv_rows(self, S, w, out) -> None: ...          # out[:n] = S w
    def factor(self, packed_gram, lam): ...              # -> factor handle; raises FactorizationError
    def trsv_pair(self, L, z) -> None: ...               # z <- L^-T L^-1 z
    def cols_solve(self, S, z, v, lam, x, accumulate: bool) -> None: ...
    def residual_cols(self, S, y, x, v, lam, r) -> tuple[float, float]: ...
    def empty(self, count: int): ...


@dataclass
class ShardedSolution:
    x_local: object
    abs_residual: float
    rel_residual: float
    refined: bool


def sharded_solve_chol(S_local, v_local, lam: float, n: int, ops: StageOps,
                       allreduce: Callable[[object], None], *, diagnostics: bool = True,
                       refine: bool = False, refine_above: float = REFINE_ABOVE_REL) -> ShardedSolution:
    """One solve of the column-sharded system; every rank calls this collectively."""
    T = n * (n + 1) // 2
    packed = ops.empty(T + n)
    ops.gram_partial(S_local, packed)
    ops.gemv_rows(S_local, v_local, packed[T:])
    allreduce(packed)                                   # sum over ranks of [G_k | u_k]
    L = ops.factor(packed[:T], lam)                     # identical on all ranks (deterministic)
    z = packed[T:]
    ops.trsv_pair(L, z)
    m_local = v_local.shape[0]
    x = ops.empty(m_local)
    ops.cols_solve(S_local, z, v_local, lam, x, accumulate=False)
    if not diagnostics:
        return ShardedSolution(x, float("nan"), float("nan"), False)
    abs_res = rel_res = float("nan")
    refined = False
    r = ops.empty(m_local)
    for rnd in range(2):
        y = ops.empty(n)
        ops.gemv_rows(S_local, x, y)
        allreduce(y)
        rr, vv = ops.residual_cols(S_local, y, x, v_local, lam, r)
        sums = ops.empty(2)
        sums[0] = rr
        sums[1] = vv
        allreduce(sums)
        rr, vv = float(sums[0]), float(sums[1])
        abs_res = float(np.sqrt(rr))
        rel_res = abs_res / max(float(np.sqrt(vv)), EPS)
        if rnd == 1 or not refine or not rel_res > refine_above:
            break
        # one correction pass with the same factor (solvers.py:183-194): r = -r; x += chol_apply(r)
        rneg = -r
        u2 = ops.empty(n)
        ops.gemv_rows(S_local, rneg, u2)
        allreduce(u2)
        ops.trsv_pair(L, u2)
        ops.cols_solve(S_local, u2, rneg, lam, x, accumulate=True)
        refined = True
    return ShardedSolution(x, abs_res, rel_res, refined)


class CudaStageOps:
    """Stage ops bound to libfisher_b200.so (device-resident torch tensors)."""

    def __init__(self, device: torch.device, n: int, m_local: int, precision: str = "auto",
                 dtype: torch.dtype = torch.float32, ctx: "_lib.Context | None" = None):
        self.device = device
        self.n = n
        # one fs_ctx per thread/stream (include/fs.h): pass a private context when several
        # ranks share a process
        self.ctx = ctx if ctx is not None else _lib.context_for(device.index, n, m_local)
        self.prec = PRECISIONS[resolve_precision(precision, dtype)]

    def _st(self):
        return _stream(self.device)

    def empty(self, count: int):
        return torch.empty(count, dtype=torch.float64, device=self.device)

    def gram_partial(self, S, out):
        n, m = S.shape
        rc = self.ctx.lib.fs_gram_packed(self.ctx.handle, _dt(S), self.prec, S.data_ptr(), n, m, S.stride(0), 0.0,
                                         out.data_ptr(), self._st())
        _check(self.ctx, rc, "fs_gram_packed")

    def gemv_rows(self, S, w, out):
        n, m = S.shape
        rc = self.ctx.lib.fs_gemv_rows(self.ctx.handle, _dt(S), S.data_ptr(), n, m, S.stride(0), w.data_ptr(),
                                       _dt(w), out.data_ptr(), self._st())
        _check(self.ctx, rc, "fs_gemv_rows")

    def factor(self, packed_gram, lam):
        n = self.n
        W = torch.empty((n, n), dtype=torch.float64, device=self.device)
        rc = self.ctx.lib.fs_unpack_lower(self.ctx.handle, packed_gram.data_ptr(), n, float(lam), W.data_ptr(), n,
                                          self._st())
        _check(self.ctx, rc, "fs_unpack_lower")
        piv = ctypes.c_int64(-1)
        rc = self.ctx.lib.fs_potrf(self.ctx.handle, W.data_ptr(), n, n, ctypes.byref(piv), self._st())
        if rc == _lib.FS_NOT_PD:
            raise FactorizationError(f"Gram matrix is not positive definite at pivot {piv.value}",
                                     pivot=int(piv.value))
        _check(self.ctx, rc, "fs_potrf")
        return W

    def trsv_pair(self, L, z):
        rc = self.ctx.lib.fs_trsv_pair(self.ctx.handle, L.data_ptr(), self.n, L.stride(0), z.data_ptr(), self._st())
        _check(self.ctx, rc, "fs_trsv_pair")

    def cols_solve(self, S, z, v, lam, x, accumulate):
        n, m = S.shape
        rc = self.ctx.lib.fs_gemv_cols_solve(self.ctx.handle, _dt(S), S.data_ptr(), n, m, S.stride(0),
                                             z.data_ptr(), v.data_ptr(), _dt(v), float(lam), int(accumulate),
                                             x.data_ptr(), self._st())
        _check(self.ctx, rc, "fs_gemv_cols_solve")

    def residual_cols(self, S, y, x, v, lam, r):
        n, m = S.shape
        sums = torch.empty(2, dtype=torch.float64, device=self.device)
        rc = self.ctx.lib.fs_residual_cols(self.ctx.handle, _dt(S), S.data_ptr(), n, m, S.stride(0), y.data_ptr(),
                                           x.data_ptr(), v.data_ptr(), _dt(v), float(lam), r.data_ptr(),
                                           sums.data_ptr(), self._st())
        _check(self.ctx, rc, "fs_residual_cols")
        rr, vv = sums.cpu().tolist()
        return rr, vv


def torch_allreduce(buf) -> None:
    """Sum-all-reduce through torch.distributed (NCCL on GPUs, gloo on CPU)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(buf)


class _DeviceBuffer:
    """Zero-copy torch view of a raw device pointer (the C ABI hands its all-reduce buffers out as
    plain pointers): __cuda_array_interface__ import, no allocation."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": (int(count),), "typestr": "<f8",
                                         "version": 3, "strides": None}


def nccl_allreduce_fn(device: torch.device, group=None):
    """An fs_allreduce_fn for fs_chol_solve: sums `count` doubles at `buf` across the ranks of
    `group` with torch.distributed (NCCL over NVLink/NVSwitch on GPUs), in place, ordered on the
    solve stream (the call is issued on torch's current stream, which is the stream passed to
    fs_chol_solve).  Returns 0 on success."""
    import torch.distributed as dist

    def fn(buf, count, user, stream):
        try:
            t = torch.as_tensor(_DeviceBuffer(buf, count), device=device)
            dist.all_reduce(t, group=group)
            return 0
        except Exception:          # surfaced by fs_chol_solve as FS_ECUDA with its message
            return 1

    return _lib.ALLREDUCE_FN(fn)


def sharded_solve_chol_fused(S_local, v_local, lam: float, *, precision: str = "auto",
                             diagnostics: bool = True, refine: int = 0, group=None) -> ShardedSolution:
    """The column-sharded solve through ONE C-ABI call per rank: the same fused kernels as the
    single-GPU path on the local shard (retile + u, tcgen05 SYRK, x + y pass, residual), with the
    C ABI's all-reduce callback doing the exchanges ([G | u], y, the norms) over NCCL.

    S_local: a CUDA tensor (validated and aligned here), a ScoreMatrix already on the device (used
    as is: validated once at construction), or a host shard (numpy / deferred host ScoreMatrix) —
    the latter goes through fs_chol_solve_host (pipelined column-chunk upload overlapped with the
    Gram) and returns x_local on the host.

    Collective-safe: validation failures of this rank's shard (non-finite entries) do not raise
    here, before the collectives — the rank joins them idle (FS_FLAG_INVALID_SHARD) and every rank
    raises ValueError together; a factorization breakdown raises FactorizationError on every rank
    (the factor is identical everywhere).  A zero-column shard (m < world) contributes nothing."""
    from .core import ScoreMatrix, _coerce_host, _to_device_tensor
    from .solvers import _pinned_out
    dev = torch.device("cuda", torch.cuda.current_device())
    host = None
    invalid = False
    S = None
    absmax = None
    if isinstance(S_local, ScoreMatrix):
        if S_local.is_uploaded or not S_local.host_origin:
            S = S_local.tensor
            dev = S.device
        else:
            host = S_local.host_array
    elif isinstance(S_local, torch.Tensor) and S_local.is_cuda:
        dev = S_local.device
        if S_local.dim() == 2 and S_local.shape[1] == 0:
            S = S_local
        else:
            S = _to_device_tensor(S_local, "score matrix", dev, validate=False)   # aligned rows (no copy when already)
            if S.dtype == torch.float32:      # the validation pass also yields the exact F16X2 row scales
                ok, absmax = _lib.row_absmax(S)
            else:
                ok = _lib.all_finite(S)
            invalid = not ok
    else:
        arr = _coerce_host(S_local, "score matrix")
        if arr.ndim == 2 and arr.shape[1] == 0:
            S = torch.empty((arr.shape[0], 0), dtype=torch.float32 if arr.dtype == np.float32 else torch.float64,
                            device=dev)
        else:
            host = ScoreMatrix(arr, defer=True).host_array        # numpy shard: validated on the device
    piv = ctypes.c_int64(-1)
    res = (ctypes.c_double * 2)(float("nan"), float("nan"))
    cb = nccl_allreduce_fn(dev, group)
    if host is not None:
        n, m = int(host.shape[0]), int(host.shape[1])
        vh = np.ascontiguousarray(v_local.detach().cpu().numpy() if isinstance(v_local, torch.Tensor)
                                  else np.asarray(v_local), dtype=host.dtype)
        prec = resolve_precision(precision, torch.float32 if host.dtype == np.float32 else torch.float64)
        flags = (_lib.FS_FLAG_RESIDUAL if diagnostics else 0) | refine_flags(prec, refine)
        ctx = _lib.context_for(dev.index, n, m)
        x = _pinned_out.get(m)
        dt = _lib.FS_F32 if host.dtype == np.float32 else _lib.FS_F64
        rc = ctx.lib.fs_chol_solve_host(ctx.handle, dt, PRECISIONS[prec], host.ctypes.data, n, m,
                                        host.strides[0] // host.itemsize, vh.ctypes.data, float(lam), x.ctypes.data,
                                        cb, None, flags, REFINE_ABOVE_REL, ctypes.byref(piv), res, _stream(dev))
        what = "fs_chol_solve_host"
    else:
        n, m = int(S.shape[0]), int(S.shape[1])
        v = v_local.to(dev).to(S.dtype).contiguous() if isinstance(v_local, torch.Tensor) else \
            torch.as_tensor(np.asarray(v_local), device=dev).to(S.dtype).contiguous()
        if m and v.numel() and not _lib.all_finite(v):
            invalid = True
        flags = _lib.FS_FLAG_INVALID_SHARD if invalid else 0
        prec = resolve_precision(precision, S.dtype)
        flags = (_lib.FS_FLAG_RESIDUAL if diagnostics else 0) | refine_flags(prec, refine) | flags
        ctx = _lib.context_for(dev.index, n, max(m, 1))
        x = torch.empty(m, dtype=torch.float64, device=dev)
        ctx.hint_row_absmax(S_local.row_absmax if isinstance(S_local, ScoreMatrix) else absmax, n)
        rc = ctx.lib.fs_chol_solve(ctx.handle, _dt(S), PRECISIONS[prec], S.data_ptr() if m else None, n, m,
                                   S.stride(0) if m else 0, v.data_ptr() if m else None, float(lam),
                                   x.data_ptr() if m else None, cb, None, flags, REFINE_ABOVE_REL,
                                   ctypes.byref(piv), res, _stream(dev))
        what = "fs_chol_solve"
    if rc == _lib.FS_NOT_PD:
        if precision == "auto" and prec != "fp64":
            # the split Gram lost definiteness (its ~2^-22 ||G|| error): every rank saw the same
            # all-reduced Gram, so every rank retries in the reference's fp64 arithmetic together
            return sharded_solve_chol_fused(S_local, v_local, lam, precision="fp64", diagnostics=diagnostics,
                                            refine=refine, group=group)
        raise FactorizationError(f"Gram matrix is not positive definite at pivot {piv.value}", pivot=int(piv.value))
    _check(ctx, rc, what)
    return ShardedSolution(x_local=x, abs_residual=float(res[0]), rel_residual=float(res[1]), refined=refine > 0)
