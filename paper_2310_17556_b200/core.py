"""Core types of the damped Fisher system, mirroring fisher_solve.core on B200.

Mirrors /root/reference/pkg/src/fisher_solve/core.py (same names, argument meaning
and errors).  Differences that make it B200-native:

* ``ScoreMatrix`` keeps the scores resident on a CUDA device (``.tensor``), in the
  caller's precision when that is float32/float64 (the reference always widens to
  float64, core.py:108-119; ints/bools still widen to float64).  Construction makes the
  private copy and validates finiteness there, as the reference does (core.py:132-142):
  a host array is uploaded and checked on the device at construction, so later changes to
  the caller's array do not reach the solve.  ``ScoreMatrix(a, defer=True)`` opts into the
  streamed host entry instead (the upload overlaps the Gram inside the solve; validation
  happens there and the caller must not modify ``a`` until the solve returns).
  ``.data`` returns a read-only host copy for code written against the reference.
* ``gram`` and ``residual`` run on the GPU through the C ABI (include/fs.h); there
  is no CPU fallback.  Complex scores go through the real embeddings of fs_embed_complex
  (no kernel ever reads complex memory as real rows).
"""

from __future__ import annotations

import enum
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

EPS = float(np.finfo(np.float64).eps)   # core.py:16


# str mixins: a member equals its value ("chol" == Method.CHOL), so the reference's own enums
# accept this package's members (fisher_solve.Method(Method.CHOL)) in code that mixes the two
class ScalarKind(str, enum.Enum):        # core.py:22-24
    REAL64 = "real64"
    REAL32 = "real32"
    COMPLEX128 = "complex128"


class Method(str, enum.Enum):            # core.py:27-35
    CHOL = "chol"
    SVD_EIGH = "eigh"
    SVD_DIRECT = "svd"
    NAIVE = "naive"
    RVB = "rvb"
    CG = "cg"


class Variant(str, enum.Enum):           # core.py:38-48
    PLAIN = "plain"
    HERMITIAN = "hermitian"
    REALPART = "realpart"


class FactorizationError(RuntimeError):  # core.py:51-60
    """A factorization broke down; ``pivot`` is the 0-based failing leading minor."""

    def __init__(self, message: str, pivot: int | None = None):
        super().__init__(message)
        self.pivot = pivot


class WorkspaceMeter:                    # core.py:63-96
    """Integer bookkeeping of scalar slots a solver allocates (device slots here)."""

    __slots__ = ("current_slots", "peak_slots")

    def __init__(self):
        self.current_slots = 0
        self.peak_slots = 0

    def alloc(self, slots: int) -> None:
        self.current_slots += int(slots)
        if self.current_slots > self.peak_slots:
            self.peak_slots = self.current_slots

    def free(self, slots: int) -> None:
        self.current_slots -= int(slots)

    def peak_bytes(self, itemsize: int = 8) -> int:
        return self.peak_slots * int(itemsize)


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.NativeLibraryError("no CUDA device: the B200 solver has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _coerce_damping(lam) -> float:       # core.py:99-105
    if isinstance(lam, bool) or not isinstance(lam, (int, float, np.integer, np.floating)):
        raise ValueError(f"damping must be a real scalar, got {type(lam).__name__}")
    lam = float(lam)
    if not np.isfinite(lam) or lam <= 0.0:
        raise ValueError(f"damping must be finite and > 0, got {lam}")
    return lam


# Pageable host arrays: the driver's own pageable copy runs at ~11 GB/s (measured, 4.1 GB in
# 374 ms).  Large ones are staged instead: worker threads copy row chunks into a ring of pinned
# buffers (numpy copyto releases the GIL, so the threads copy in parallel) while the previous
# chunk's DMA to the device runs.
_STAGE_MIN_BYTES = 64 << 20
_STAGE_CHUNK_BYTES = 64 << 20
_STAGE_BUFFERS = 3
_stage_state: dict = {}


def _stage_pool():
    if "pool" not in _stage_state:
        import concurrent.futures
        import os
        workers = int(os.environ.get("FS_STAGE_WORKERS", "0")) or max(1, min(8, (os.cpu_count() or 2) - 1))
        _stage_state["pool"] = concurrent.futures.ThreadPoolExecutor(max_workers=workers)
        _stage_state["workers"] = workers
        _stage_state["bufs"] = [torch.empty(_STAGE_CHUNK_BYTES, dtype=torch.uint8, pin_memory=True)
                                for _ in range(_STAGE_BUFFERS)]
        _stage_state["events"] = [None] * _STAGE_BUFFERS    # last DMA reading each buffer (any call)
        import threading
        _stage_state["lock"] = threading.Lock()
    return _stage_state["pool"], _stage_state["workers"], _stage_state["bufs"]


def _upload_staged(src: torch.Tensor, dst: torch.Tensor) -> None:
    """dst (CUDA, rows of a 2-D view) <- src (pageable CPU, C-contiguous 2-D), row chunks through
    pinned staging buffers; ordered on the current stream, returns once the last chunk is queued."""
    pool, workers, bufs = _stage_pool()
    rows, cols = int(src.shape[0]), int(src.shape[1])
    row_bytes = cols * src.element_size()
    per = max(1, _STAGE_CHUNK_BYTES // row_bytes)
    if per * row_bytes > _STAGE_CHUNK_BYTES:        # one row larger than a buffer: plain copy
        dst.copy_(src)
        return
    stream = torch.cuda.current_stream(dst.device)
    src_np = src.numpy()
    with _stage_state["lock"]:
        _staged_chunks(pool, workers, bufs, _stage_state["events"], src, src_np, dst, rows, cols, row_bytes, per,
                       stream)


def _staged_chunks(pool, workers, bufs, events, src, src_np, dst, rows, cols, row_bytes, per, stream):
    for i, r0 in enumerate(range(0, rows, per)):
        r1 = min(rows, r0 + per)
        k = i % len(bufs)
        if events[k] is not None:
            events[k].synchronize()                 # the DMA that last read this buffer is done
        view = bufs[k][: (r1 - r0) * row_bytes].view(src.dtype).view(r1 - r0, cols)
        # split the chunk's bytes (contiguous rows) evenly over the workers, not whole rows: a 64 MB
        # chunk of 4 MB rows has only 16 rows
        vflat = view.numpy().reshape(-1)
        sflat = src_np[r0:r1].reshape(-1)
        step = -(-vflat.size // workers)
        step = -(-step // 1024) * 1024            # 4-8 KB aligned pieces
        futs = [pool.submit(np.copyto, vflat[a:a + step], sflat[a:a + step]) for a in range(0, vflat.size, step)]
        for f in futs:
            f.result()
        dst[r0:r1].copy_(view, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        events[k] = ev


def _to_device_tensor(a, name: str, device, force_copy: bool = False, validate: bool = True) -> torch.Tensor:
    """Coerce to a float32/float64 (or complex64/complex128) CUDA tensor and validate finiteness
    (core.py:108-119).

    2-D inputs get unit column stride and 16-byte aligned rows (padded leading dimension);
    ``force_copy`` guarantees the result does not alias ``a`` (the reference freezes a copy).
    Host arrays are always copied (uploaded), so the result never aliases them.
    """
    if isinstance(a, torch.Tensor):
        t = a
        if t.is_complex():
            if t.dtype not in (torch.complex64, torch.complex128):
                t = t.to(torch.complex128)
        elif t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
    else:
        arr = _coerce_host(a, name)
        with warnings.catch_warnings():      # read-only arrays (e.g. another ScoreMatrix's .data)
            warnings.simplefilter("ignore", UserWarning)
            t = torch.from_numpy(arr)
    dev = device if device is not None else (t.device if t.is_cuda else default_device())
    if t.dim() == 2 and t.shape[1] > 0:
        # rows start on 16-byte boundaries (TMA / vector-load requirement); pad columns are never read
        per16 = max(1, 16 // t.element_size())
        ld = -(-t.shape[1] // per16) * per16
        if force_copy or not (t.is_cuda and t.device == dev and t.stride(1) == 1 and t.stride(0) % per16 == 0
                              and t.data_ptr() % 16 == 0):
            buf = torch.empty((t.shape[0], ld), dtype=t.dtype, device=dev)
            if (not t.is_cuda and not t.is_pinned() and t.is_contiguous() and not t.is_complex()
                    and t.numel() * t.element_size() >= _STAGE_MIN_BYTES):
                _upload_staged(t, buf[:, : t.shape[1]])
                t = buf[:, : t.shape[1]]
            else:
                t = buf[:, : t.shape[1]].copy_(t, non_blocking=True)
    else:
        src_ptr = a.data_ptr() if isinstance(a, torch.Tensor) else None
        t = t.to(dev, non_blocking=True).contiguous()
        if force_copy and src_ptr is not None and t.data_ptr() == src_ptr:
            t = t.clone()
    if validate and t.numel() and not _lib.all_finite(t):
        raise ValueError(f"{name} must contain only finite entries")
    return t


def _coerce_host(a, name: str) -> np.ndarray:
    """numpy side of core.py:108-119: numeric dtype -> C-contiguous float32/float64 (complex64 /
    complex128 for complex input); no copy when it already is one."""
    arr = np.asarray(a)
    if np.iscomplexobj(arr):      # complex scores: complex64 kept, else complex128
        return np.ascontiguousarray(arr if arr.dtype in (np.complex64, np.complex128) else arr.astype(np.complex128))
    if not (np.issubdtype(arr.dtype, np.number) or arr.dtype == np.bool_):
        raise ValueError(f"{name} must be numeric, got dtype {arr.dtype}")
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    return np.ascontiguousarray(arr)


_HOST_DTYPES = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
                np.dtype(np.complex64): torch.complex64, np.dtype(np.complex128): torch.complex128}


class ScoreMatrix:
    """Dense n-by-m score matrix, one sample per row (core.py:122-162).

    Construction validates and freezes a private copy like the reference (core.py:132-142): a
    CUDA tensor is copied onto an aligned device buffer, a host array (numpy, lists) is uploaded
    to one; non-finite entries raise ValueError here, and the caller's array is neither frozen
    nor read again.

    ``defer=True`` (host arrays only) keeps the array on the host until the first solve, which
    streams it to the GPU in column chunks overlapped with the Gram (fs_chol_solve_host) and
    checks finiteness there — the fastest host-to-answer path, at the cost of the reference's
    construction-time checks: the caller must not modify the array until the solve returns.
    """

    def __init__(self, data, device=None, *, defer: bool = False):
        src = data
        self._host = None
        self._t = None
        self._src = None
        self._absmax = None
        self._device = device
        if isinstance(src, torch.Tensor):
            t = self._validated(_to_device_tensor(data, "score matrix", device, force_copy=src.is_cuda,
                                                  validate=False))
            shape = tuple(t.shape)
            self._t = t
        else:
            arr = _coerce_host(data, "score matrix")
            shape = arr.shape
            if len(shape) == 2 and shape[0] >= 1 and shape[1] >= 1:
                if defer and not np.iscomplexobj(arr):
                    self._src = arr
                else:
                    self._t = self._validated(_to_device_tensor(arr, "score matrix", device, validate=False))
        if len(shape) != 2:
            raise ValueError(f"score matrix must be 2-D, got shape {shape}")
        if shape[0] < 1 or shape[1] < 1:
            raise ValueError(f"score matrix needs at least one row and column, got {shape}")
        self._shape = (int(shape[0]), int(shape[1]))
        # numpy in -> numpy out (drop-in semantics); CUDA tensor in -> CUDA tensor out
        self.host_origin = not (isinstance(src, torch.Tensor) and src.is_cuda)

    def _validated(self, t: torch.Tensor) -> torch.Tensor:
        """Finiteness check on the device (core.py:108-119); for float32 scores the same pass keeps
        each row's max |S_i| — the exact F16X2 row scales of every later solve (fs_row_absmax)."""
        if t.numel() == 0:
            return t
        if t.dim() == 2 and t.dtype == torch.float32:
            ok, self._absmax = _lib.row_absmax(t)
        else:
            ok = _lib.all_finite(t)
        if not ok:
            raise ValueError("score matrix must contain only finite entries")
        return t

    @property
    def row_absmax(self) -> torch.Tensor | None:
        """Per-row max |S_i| of float32 scores (device), computed at validation; None otherwise."""
        return self._absmax

    @classmethod
    def _owned(cls, t: torch.Tensor, host_origin: bool = False) -> "ScoreMatrix":
        """Wrap a device tensor this package produced (aligned rows, finite): no copy, no check."""
        sm = cls.__new__(cls)
        sm._host = None
        sm._src = None
        sm._absmax = None
        sm._t = t
        sm._device = t.device
        sm._shape = (int(t.shape[0]), int(t.shape[1]))
        sm.host_origin = host_origin
        return sm

    @property
    def is_uploaded(self) -> bool:
        return self._t is not None

    @property
    def host_array(self) -> np.ndarray | None:
        """The C-contiguous host array of a deferred (``defer=True``) matrix not uploaded yet."""
        return None if self._t is not None else self._src

    @property
    def tensor(self) -> torch.Tensor:
        if self._t is None:
            self._t = self._validated(_to_device_tensor(self._src, "score matrix", self._device, validate=False))
            self._src = None
        return self._t

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            h = np.array(self._src) if self._t is None else self._t.cpu().numpy()
            h = np.ascontiguousarray(h)
            h.flags.writeable = False
            self._host = h
        return self._host

    @property
    def n(self) -> int:
        return self._shape[0]

    @property
    def m(self) -> int:
        return self._shape[1]

    @property
    def shape(self) -> tuple[int, int]:
        return self._shape

    @property
    def is_complex(self) -> bool:
        return self.dtype in (torch.complex64, torch.complex128)

    @property
    def dtype(self) -> torch.dtype:
        if self._t is not None:
            return self._t.dtype
        return _HOST_DTYPES.get(self._src.dtype, torch.float64)

    @property
    def device(self) -> torch.device:
        if self._t is not None:
            return self._t.device
        return self._device if self._device is not None else default_device()

    @property
    def scalar_kind(self) -> ScalarKind:
        if self.is_complex:
            return ScalarKind.COMPLEX128
        return ScalarKind.REAL64 if self.dtype == torch.float64 else ScalarKind.REAL32

    @property
    def real_dtype(self) -> torch.dtype:
        """The real scalar type of the scores (float32 for complex64, float64 for complex128)."""
        return {torch.complex64: torch.float32, torch.complex128: torch.float64}.get(self.dtype, self.dtype)


def as_scores(S) -> "ScoreMatrix":
    """A ScoreMatrix of this package from one, from a reference ``fisher_solve.ScoreMatrix`` (any
    object with a ``.data`` array, core.py:122-162) or from raw data — so code holding the
    reference's objects can call the B200 entry points unchanged."""
    if isinstance(S, ScoreMatrix):
        return S
    if not isinstance(S, (np.ndarray, torch.Tensor, list, tuple)) and hasattr(S, "data"):
        return ScoreMatrix(S.data)
    return ScoreMatrix(S)


def as_system(system) -> "DampedSystem":
    """A DampedSystem of this package from one or from a reference ``fisher_solve.DampedSystem``
    (``.S``, ``.lam``, ``.v``, core.py:165-203)."""
    if isinstance(system, DampedSystem):
        return system
    if all(hasattr(system, a) for a in ("S", "lam", "v")):
        return DampedSystem(as_scores(system.S), system.lam, system.v)
    raise ValueError(f"expected a DampedSystem, got {type(system).__name__}")


class DampedSystem:
    """The system (S^T S + lam I) x = v (core.py:165-203); v lives beside S in S's dtype.

    v is validated (1-D, length m, finite, real when S is real) and copied at construction, like
    the reference's frozen copy (core.py:179-195)."""

    def __init__(self, S: ScoreMatrix, lam, v):
        S = as_scores(S)
        self.S = S
        self.lam = _coerce_damping(lam)
        v_complex = v.is_complex() if isinstance(v, torch.Tensor) else np.iscomplexobj(np.asarray(v))
        if v_complex and not S.is_complex:
            raise ValueError("real score matrix with complex right-hand side")
        self._v = None
        self._vh = None
        self._host_v = None
        if S.host_array is not None and not (isinstance(v, torch.Tensor) and v.is_cuda):
            # deferred host system: v stays on the host beside S (validated and copied here)
            vh = _coerce_host(v.numpy() if isinstance(v, torch.Tensor) else v, "right-hand side")
            if vh.ndim != 1:
                raise ValueError(f"right-hand side must be 1-D, got shape {vh.shape}")
            if vh.shape[0] != S.m:
                raise ValueError(f"right-hand side length {vh.shape[0]} does not match parameter count {S.m}")
            if not np.isfinite(vh).all():
                raise ValueError("right-hand side must contain only finite entries")
            self._vh = np.array(vh, dtype=np.float32 if S.dtype == torch.float32 else np.float64, copy=True)
            return
        t = _to_device_tensor(v, "right-hand side", S.tensor.device,
                              force_copy=isinstance(v, torch.Tensor) and v.is_cuda)
        if t.dim() != 1:
            raise ValueError(f"right-hand side must be 1-D, got shape {tuple(t.shape)}")
        if t.shape[0] != S.m:
            raise ValueError(f"right-hand side length {t.shape[0]} does not match parameter count {S.m}")
        if S.is_complex:
            # complex scores: v keeps its own kind (the real-part variant needs a
            # real v), in the scores' precision
            self._v = t.to(S.dtype if t.is_complex() else S.real_dtype)
        else:
            self._v = t.to(S.dtype)

    @property
    def host_v(self) -> np.ndarray | None:
        """v on the host (S's dtype) while a deferred system has not been uploaded."""
        return self._vh if self._v is None else None

    @property
    def v_tensor(self) -> torch.Tensor:
        if self._v is None:
            self._v = torch.from_numpy(self._vh).to(self.S.tensor.device)
        return self._v

    @property
    def v(self) -> np.ndarray:
        if self._host_v is None:
            h = self._vh.copy() if self._v is None else self._v.cpu().numpy()
            h.flags.writeable = False
            self._host_v = h
        return self._host_v

    @property
    def n(self) -> int:
        return self.S.n

    @property
    def m(self) -> int:
        return self.S.m


@dataclass(frozen=True)
class Solution:                          # core.py:206-223
    x: object          # numpy float64 (host systems) or a CUDA float64 tensor (device systems)
    method: Method
    abs_residual: float
    rel_residual: float
    wall_seconds: float
    iterations: int | None = None
    converged: bool = True
    precision: str = "fp64"


def _dt(t: torch.Tensor) -> int:
    """fs_dtype of a REAL device array; complex data never reaches a real kernel (ValueError)."""
    if t.dtype == torch.float64:
        return _lib.FS_F64
    if t.dtype == torch.float32:
        return _lib.FS_F32
    raise ValueError(f"this kernel takes real float32/float64 data, got {t.dtype}"
                     + (" (complex scores go through the real embeddings)" if t.is_complex() else ""))


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _check(ctx, rc: int, what: str):
    if rc == _lib.FS_OK:
        return
    msg = f"{what}: {ctx.last_error()} (status {rc})"
    if rc in (_lib.FS_EINVAL, _lib.FS_EUNSUPPORTED):
        raise ValueError(msg)
    raise _lib.NativeLibraryError(msg)


PRECISIONS = {"fp64": _lib.FS_PREC_FP64, "tf32x3": _lib.FS_PREC_TF32X3, "f16x2": _lib.FS_PREC_F16X2,
              "auto": _lib.FS_PREC_AUTO}


def resolve_precision(precision: str, dtype: torch.dtype) -> str:
    """fp64: exact fp64 products.  f16x2 (default for float32 scores): each element split into two
    row-scaled fp16 planes (22 significant bits), kind::f16 tensor-core Gram.  tf32x3: the
    kind::tf32 three-product split.  Both fp32 modes carry the stated 4 u32 sigma^2/lam bound."""
    if precision not in PRECISIONS:
        raise ValueError(f"unknown precision {precision!r}; expected one of {sorted(PRECISIONS)}")
    if precision == "auto":
        return "f16x2" if dtype == torch.float32 else "fp64"
    if precision in ("tf32x3", "f16x2") and dtype != torch.float32:
        raise ValueError(f"precision {precision!r} needs float32 scores")
    return precision


def gram_packed(S: ScoreMatrix, lam: float, precision: str = "auto") -> torch.Tensor:
    """Packed lower W = S S^T + lam I on the device (fp64, length n(n+1)/2); real scores only
    (complex scores: ``gram`` returns the Hermitian S S^H + lam I)."""
    t = S.tensor
    n, m = S.n, S.m
    dt = _dt(t)
    prec = resolve_precision(precision, t.dtype)
    ctx = _lib.context_for(t.device.index, n, m)
    out = torch.empty(n * (n + 1) // 2, dtype=torch.float64, device=t.device)
    hint_scales(ctx, S)
    rc = ctx.lib.fs_gram_packed(ctx.handle, dt, PRECISIONS[prec], t.data_ptr(), n, m, t.stride(0),
                                float(lam), out.data_ptr(), _stream(t.device))
    _check(ctx, rc, "fs_gram_packed")
    return out


def hint_scales(ctx, S: "ScoreMatrix") -> None:
    """Exact F16X2 row scales for the next call on ctx when the scores carry their row maxima."""
    ctx.hint_row_absmax(S.row_absmax if isinstance(S, ScoreMatrix) else None, S.n)


def gram_hermitian_device(S: ScoreMatrix, lam: float, precision: str = "auto") -> torch.Tensor:
    """W = S S^H + lam I for complex scores, an n x n complex128 CUDA tensor, exactly Hermitian
    (core.py:279-290).  The Gram of C = [Re S; Im S] (2n x m, fs_embed_complex kind 0) holds
    Re S Re S^T + Im S Im S^T (the real part) and Im S Re S^T - Re S Im S^T (the imaginary part)
    in its blocks; fs_hermitian_gram combines them, mirrors with conjugation and adds lam."""
    if not S.is_complex:
        raise ValueError("gram_hermitian_device expects complex scores")
    n = S.n
    C = embed_complex(S, 0)
    G2 = gram_packed(C, 0.0, precision)
    dev = G2.device
    W = torch.empty((n, n), dtype=torch.complex128, device=dev)
    ctx = _lib.context_for(dev.index, 2 * n, S.m)
    rc = ctx.lib.fs_hermitian_gram(ctx.handle, G2.data_ptr(), n, float(lam), W.data_ptr(), n, _stream(dev))
    _check(ctx, rc, "fs_hermitian_gram")
    return W


def gram(S: ScoreMatrix, lam: float, meter: WorkspaceMeter | None = None, precision: str = "auto") -> np.ndarray:
    """Damped Gram matrix W = S S^T + lam I (S S^H for complex S), n-by-n, exactly symmetric /
    Hermitian (core.py:270-290)."""
    lam = _coerce_damping(lam)
    S = as_scores(S)
    n = S.n
    if S.is_complex:
        if meter is not None:
            meter.alloc(2 * S.n * S.m)          # the embedded copy [Re S; Im S]
            meter.alloc(2 * n * (2 * n + 1))
            meter.free(2 * S.n * S.m)
        W = gram_hermitian_device(S, lam, precision).cpu().numpy()
        if meter is not None:
            meter.alloc(2 * n * n)
            meter.free(2 * n * (2 * n + 1))
        return W
    if meter is not None:
        meter.alloc(n * (n + 1) // 2)
    packed = gram_packed(S, lam, precision).cpu().numpy()
    W = np.zeros((n, n))
    W[np.tril_indices(n)] = packed
    W = W + np.tril(W, -1).T   # mirror: exactly symmetric by construction
    if meter is not None:
        meter.alloc(n * n)
        meter.free(n * (n + 1) // 2)
    return W


def residual_device(system: DampedSystem, x: torch.Tensor) -> tuple[float, float]:
    """||(S^T S + lam I) x - v|| and its relative value, fp64 on the device (core.py:307-322)."""
    S = system.S.tensor
    n, m = system.n, system.m
    ctx = _lib.context_for(S.device.index, n, m)
    st = _stream(S.device)
    y = torch.empty(n, dtype=torch.float64, device=S.device)
    sums = torch.empty(2, dtype=torch.float64, device=S.device)
    rc = ctx.lib.fs_gemv_rows(ctx.handle, _dt(S), S.data_ptr(), n, m, S.stride(0), x.data_ptr(), _lib.FS_F64,
                              y.data_ptr(), st)
    _check(ctx, rc, "fs_gemv_rows")
    v = system.v_tensor
    rc = ctx.lib.fs_residual_cols(ctx.handle, _dt(S), S.data_ptr(), n, m, S.stride(0), y.data_ptr(), x.data_ptr(),
                                  v.data_ptr(), _dt(v), system.lam, None, sums.data_ptr(), st)
    _check(ctx, rc, "fs_residual_cols")
    rr, vv = sums.cpu().tolist()
    abs_res = float(np.sqrt(rr))
    return abs_res, abs_res / max(float(np.sqrt(vv)), EPS)


def embed_complex(S: ScoreMatrix, kind: int) -> ScoreMatrix:
    """Real stand-ins for complex scores on the device (fs_embed_complex):
    kind 0 -> C = [Re S; Im S] (sr.py:61-70), kind 1 -> [[Re S, -Im S], [Im S, Re S]]."""
    if not S.is_complex:
        raise ValueError("embed_complex expects a complex score matrix")
    t = S.tensor
    n, m = S.n, S.m
    rdt = S.real_dtype
    cols = m if kind == 0 else 2 * m
    per16 = 16 // torch.empty((), dtype=rdt).element_size()
    ld = -(-cols // per16) * per16
    buf = torch.empty((2 * n, ld), dtype=rdt, device=t.device)
    ctx = _lib.context_for(t.device.index, n, m)
    rc = ctx.lib.fs_embed_complex(ctx.handle, kind, _lib.FS_F64 if rdt == torch.float64 else _lib.FS_F32,
                                  t.data_ptr(), n, m, t.stride(0), buf.data_ptr(), ld, _stream(t.device))
    _check(ctx, rc, "fs_embed_complex")
    return ScoreMatrix._owned(buf[:, :cols])


def stack_complex_vector(v: torch.Tensor, real_dtype: torch.dtype) -> torch.Tensor:
    """[Re v; Im v] (2m), the right-hand side of the real representation."""
    if v.is_complex():
        return torch.cat([v.real, v.imag]).to(real_dtype).contiguous()
    return torch.cat([v.to(real_dtype), torch.zeros_like(v, dtype=real_dtype)]).contiguous()


def residual(system: DampedSystem, x, variant: Variant = Variant.PLAIN) -> tuple[float, float]:
    """Absolute and relative residual of x (core.py:307-322), evaluated on the GPU.

    HERMITIAN (S^H S + lam I) and REALPART (Re[S^H S] + lam I) are evaluated through the real
    representation / the stacked real matrix (fs_embed_complex): the same norms."""
    system = as_system(system)
    if not isinstance(variant, Variant):
        variant = _as_variant(variant)
    if variant is not Variant.PLAIN:
        if not system.S.is_complex:
            raise ValueError(f"variant {variant.value} expects complex scores")
        dev = system.S.tensor.device
        xt = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
        xt = xt.to(dev)
        if xt.dim() != 1 or xt.shape[0] != system.m:
            raise ValueError(f"solution vector has shape {tuple(xt.shape)}, expected ({system.m},)")
        if variant is Variant.HERMITIAN:
            inner = DampedSystem(embed_complex(system.S, 1), system.lam,
                                 stack_complex_vector(system.v_tensor, system.S.real_dtype))
            return residual_device(inner, stack_complex_vector(xt, torch.float64))
        if system.v_tensor.is_complex() or xt.is_complex():
            raise ValueError("the real-part operator needs a real right-hand side and solution")
        inner = DampedSystem(embed_complex(system.S, 0), system.lam, system.v_tensor)
        return residual_device(inner, xt.to(torch.float64).contiguous())
    if system.S.is_complex:
        return _residual_plain_complex(system, x)
    if isinstance(x, torch.Tensor):
        xt = x.to(system.S.tensor.device)
    else:
        xa = np.asarray(x)
        if xa.ndim != 1 or xa.shape[0] != system.m:
            raise ValueError(f"solution vector has shape {xa.shape}, expected ({system.m},)")
        xt = torch.from_numpy(np.ascontiguousarray(xa)).to(system.S.tensor.device)
    if xt.is_complex():
        # real operator, complex x: ||A Re x - v||^2 + ||A Im x||^2 (core.py:296-297 on complex x)
        if xt.dim() != 1 or xt.shape[0] != system.m:
            raise ValueError(f"solution vector has shape {tuple(xt.shape)}, expected ({system.m},)")
        a_re, _ = residual_device(system, xt.real.to(torch.float64).contiguous())
        zero = DampedSystem(system.S, system.lam, torch.zeros_like(system.v_tensor))
        a_im, _ = residual_device(zero, xt.imag.to(torch.float64).contiguous())
        abs_res = float(np.hypot(a_re, a_im))
        return abs_res, abs_res / max(float(torch.linalg.vector_norm(system.v_tensor.double())), EPS)
    xt = xt.to(torch.float64).contiguous()
    if xt.dim() != 1 or xt.shape[0] != system.m:
        raise ValueError(f"solution vector has shape {tuple(xt.shape)}, expected ({system.m},)")
    return residual_device(system, xt)


def _as_variant(variant) -> Variant:
    """Variant from this package's enum, the reference's (same values) or its string value."""
    try:
        return Variant(getattr(variant, "value", variant))
    except ValueError:
        raise ValueError(f"unknown operator variant: {variant!r}") from None


def _residual_plain_complex(system: DampedSystem, x) -> tuple[float, float]:
    """PLAIN variant on complex scores: ||S^T (S x) + lam x - v|| without conjugation, as
    core.py:296-297 evaluates it for complex A.  With rho(S) = [[Re S, -Im S], [Im S, Re S]]
    (fs_embed_complex kind 1): rho(S) [Re x; Im x] = [Re Sx; Im Sx], and rho(S)^T applied to
    [Re t; -Im t] gives [Re S^T t; -Im S^T t]; so with y' = [Re Sx; -Im Sx], x' = [Re x; -Im x]
    and v' = [Re v; -Im v], fs_residual_cols forms [Re r; -Im r] and the same norms."""
    S = system.S
    dev = S.tensor.device
    xt = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(np.asarray(x)))
    xt = xt.to(dev)
    if xt.dim() != 1 or xt.shape[0] != system.m:
        raise ValueError(f"solution vector has shape {tuple(xt.shape)}, expected ({system.m},)")
    n, m = S.n, S.m
    E = embed_complex(S, 1).tensor
    xhat = stack_complex_vector(xt, torch.float64)
    ctx = _lib.context_for(dev.index, 2 * n, 2 * m)
    st = _stream(dev)
    y = torch.empty(2 * n, dtype=torch.float64, device=dev)
    rc = ctx.lib.fs_gemv_rows(ctx.handle, _dt(E), E.data_ptr(), 2 * n, 2 * m, E.stride(0), xhat.data_ptr(),
                              _lib.FS_F64, y.data_ptr(), st)
    _check(ctx, rc, "fs_gemv_rows")
    y[n:].neg_()
    xflip = xhat.clone()
    xflip[m:].neg_()
    vflip = stack_complex_vector(system.v_tensor, torch.float64)
    vflip[m:].neg_()
    sums = torch.empty(2, dtype=torch.float64, device=dev)
    rc = ctx.lib.fs_residual_cols(ctx.handle, _dt(E), E.data_ptr(), 2 * n, 2 * m, E.stride(0), y.data_ptr(),
                                  xflip.data_ptr(), vflip.data_ptr(), _lib.FS_F64, system.lam, None,
                                  sums.data_ptr(), st)
    _check(ctx, rc, "fs_residual_cols")
    rr, vv = sums.cpu().tolist()
    abs_res = float(np.sqrt(rr))
    return abs_res, abs_res / max(float(np.sqrt(vv)), EPS)
