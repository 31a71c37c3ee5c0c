"""ctypes binding of libfisher_b200.so (the C ABI declared in include/fs.h).

There is no CPU fallback: importing the solver entry points without the built
library, or calling them without a CUDA device, raises immediately.
"""

from __future__ import annotations

import ctypes
import os
import threading

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfisher_b200.so")

FS_OK, FS_EINVAL, FS_NOT_PD, FS_ECUDA, FS_ENOMEM, FS_EUNSUPPORTED, FS_ENOCONV = range(7)
FS_F32, FS_F64 = 0, 1
FS_PREC_FP64, FS_PREC_TF32X3, FS_PREC_AUTO, FS_PREC_F16X2 = 0, 1, 2, 3
FS_FLAG_RESIDUAL, FS_FLAG_REFINE, FS_FLAG_REFINE_Z, FS_FLAG_INVALID_SHARD = 1, 2, 4, 0x10000
PROF_STAGES = ("gram", "gemv_sv", "allreduce", "potrf", "trsv", "gemv_stz", "residual", "refine")

_c_int64 = ctypes.c_int64
_vp = ctypes.c_void_p
_dp = ctypes.POINTER(ctypes.c_double)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, _vp, _c_int64, _vp, _vp)

# name -> (restype, argtypes); must match include/fs.h exactly
SIGNATURES = {
    "fs_version": (ctypes.c_char_p, []),
    "fs_ctx_create": (ctypes.c_int, [ctypes.POINTER(_vp), ctypes.c_int, _c_int64, _c_int64]),
    "fs_ctx_destroy": (None, [_vp]),
    "fs_last_error": (ctypes.c_char_p, [_vp]),
    "fs_workspace_bytes": (ctypes.c_size_t, [_c_int64, _c_int64, ctypes.c_int, ctypes.c_int]),
    "fs_launch_count": (_c_int64, [_vp]),
    "fs_profile_enable": (ctypes.c_int, [_vp, ctypes.c_int]),
    "fs_profile_read": (ctypes.c_int, [_vp, _dp, ctypes.c_int]),
    "fs_gram_packed": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _c_int64, _c_int64, _c_int64,
                                      ctypes.c_double, _vp, _vp]),
    "fs_gemv_rows": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _c_int64, _c_int64, _c_int64, _vp, ctypes.c_int,
                                    _vp, _vp]),
    "fs_unpack_lower": (ctypes.c_int, [_vp, _vp, _c_int64, ctypes.c_double, _vp, _c_int64, _vp]),
    "fs_potrf": (ctypes.c_int, [_vp, _vp, _c_int64, _c_int64, ctypes.POINTER(_c_int64), _vp]),
    "fs_potrf_async": (ctypes.c_int, [_vp, _vp, _c_int64, _c_int64, _vp]),
    "fs_status_read": (_c_int64, [_vp, _vp]),
    "fs_trsv_pair": (ctypes.c_int, [_vp, _vp, _c_int64, _c_int64, _vp, _vp]),
    "fs_gemv_cols_solve": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _c_int64, _c_int64, _c_int64, _vp, _vp,
                                          ctypes.c_int, ctypes.c_double, ctypes.c_int, _vp, _vp]),
    "fs_residual_cols": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _c_int64, _c_int64, _c_int64, _vp, _vp, _vp,
                                        ctypes.c_int, ctypes.c_double, _vp, _vp, _vp]),
    "fs_chol_solve": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _c_int64, _c_int64, _c_int64, _vp,
                                     ctypes.c_double, _vp, ALLREDUCE_FN, _vp, ctypes.c_int, ctypes.c_double,
                                     ctypes.POINTER(_c_int64), _dp, _vp]),
    "fs_syevj_packed": (ctypes.c_int, [_vp, _vp, _c_int64, _vp, _vp, _c_int64, ctypes.POINTER(ctypes.c_int), _vp]),
    "fs_eigh_solve": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _c_int64, _c_int64, _c_int64, _vp,
                                     ctypes.c_double, ctypes.c_double, _vp, ALLREDUCE_FN, _vp, ctypes.c_int,
                                     ctypes.POINTER(_c_int64), _dp, _vp]),
    "fs_embed_complex": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _c_int64, _c_int64, _c_int64, _vp,
                                        _c_int64, _vp]),
    "fs_hermitian_gram": (ctypes.c_int, [_vp, _vp, _c_int64, ctypes.c_double, _vp, _c_int64, _vp]),
    "fs_apply_rows": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _c_int64, _c_int64, _c_int64, _vp, _c_int64, _c_int64,
                                     _vp, _c_int64, _vp]),
    "fs_apply_rows_lower": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _c_int64, _c_int64, _c_int64, _vp, _c_int64,
                                           _c_int64, _vp, _c_int64, _vp]),
    "fs_heevj_packed": (ctypes.c_int, [_vp, _vp, _c_int64, _vp, _vp, _c_int64, ctypes.POINTER(ctypes.c_int), _vp]),
    "fs_tri_inverse": (ctypes.c_int, [_vp, _vp, _c_int64, _c_int64, _vp, _c_int64, _vp]),
    "fs_jacobi_svd": (ctypes.c_int, [_vp, _vp, _c_int64, _c_int64, _vp, _vp, _c_int64, _vp, _c_int64,
                                     ctypes.POINTER(ctypes.c_int), _vp]),
    "fs_factor_solve": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _c_int64, _c_int64, _c_int64, _vp, ctypes.c_double,
                                       _vp, _c_int64, _vp, _c_int64, _vp, ctypes.c_int, _dp, _vp]),
    "fs_row_absmax": (ctypes.c_int, [ctypes.c_int, _vp, _c_int64, _c_int64, _c_int64, _vp, _vp]),
    "fs_set_row_absmax": (ctypes.c_int, [_vp, _vp, _c_int64]),
    "fs_fallback_count": (_c_int64, [_vp]),
    "fs_gram_splits": (ctypes.c_int, [_vp, _c_int64, _c_int64, ctypes.c_int]),
    "fs_all_finite": (ctypes.c_int, [ctypes.c_int, _vp, _c_int64, _c_int64, _c_int64, _vp]),
    "fs_chol_solve_host": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _c_int64, _c_int64, _c_int64, _vp,
                                          ctypes.c_double, _vp, ALLREDUCE_FN, _vp, ctypes.c_int, ctypes.c_double,
                                          ctypes.POINTER(_c_int64), _dp, _vp]),
}

_lib = None
_lock = threading.Lock()


class NativeLibraryError(RuntimeError):
    """The CUDA extension is missing or unusable; there is deliberately no fallback."""


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes library with typed signatures."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{path} is missing: build it with `python -m paper_2310_17556_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class Context:
    """Owns one fs_ctx (device workspaces) sized for n <= n_max, m <= m_max."""

    def __init__(self, device: int, n_max: int, m_max: int):
        self.lib = load()
        self.device = int(device)
        self.n_max = int(n_max)
        self.m_max = int(m_max)
        h = _vp()
        rc = self.lib.fs_ctx_create(ctypes.byref(h), self.device, self.n_max, self.m_max)
        if rc != FS_OK:
            raise NativeLibraryError(f"fs_ctx_create failed with status {rc} (n_max={n_max}, m_max={m_max})")
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            self.lib.fs_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    def last_error(self) -> str:
        return (self.lib.fs_last_error(self.handle) or b"").decode()

    def launches(self) -> int:
        return int(self.lib.fs_launch_count(self.handle))

    def profile(self, on: bool = True) -> None:
        self.lib.fs_profile_enable(self.handle, 1 if on else 0)

    def fallbacks(self) -> int:
        return int(self.lib.fs_fallback_count(self.handle))

    def hint_row_absmax(self, absmax, n: int) -> None:
        """Exact F16X2 row scales for the next solve / Gram on this context (fs_set_row_absmax)."""
        self.lib.fs_set_row_absmax(self.handle, None if absmax is None else absmax.data_ptr(), int(n))

    def stage_ms(self) -> dict:
        buf = (ctypes.c_double * len(PROF_STAGES))()
        self.lib.fs_profile_read(self.handle, buf, len(PROF_STAGES))
        return dict(zip(PROF_STAGES, list(buf)))


_contexts: dict[int, Context] = {}


def all_finite(t) -> bool:
    """True when every entry of the CUDA tensor t (1-D, or 2-D row-major with unit column stride;
    complex via its real view) is finite — fs_all_finite, one device pass, no temporaries
    (replaces torch.isfinite(t).all(), which materialised |t| and a bool copy of S)."""
    import torch
    if t.is_complex():
        r = torch.view_as_real(t)
        rows, cols, ld = (1, 2 * t.numel(), 2 * t.numel()) if t.dim() == 1 else (t.shape[0], 2 * t.shape[1], 2 * t.stride(0))
        base, dt = r, (FS_F64 if r.dtype == torch.float64 else FS_F32)
    else:
        rows, cols, ld = (1, t.numel(), t.numel()) if t.dim() == 1 else (t.shape[0], t.shape[1], t.stride(0))
        base, dt = t, (FS_F64 if t.dtype == torch.float64 else FS_F32)
    if t.dim() == 2 and t.stride(1) != 1 or t.dim() == 1 and t.stride(0) != 1:
        raise ValueError("all_finite needs unit column stride")
    lib = load()
    with torch.cuda.device(t.device):
        rc = lib.fs_all_finite(dt, base.data_ptr(), rows, cols, ld, torch.cuda.current_stream(t.device).cuda_stream)
    if rc not in (0, 1):
        raise NativeLibraryError(f"fs_all_finite failed (status {rc})")
    return rc == 0


def row_absmax(t):
    """(finite, absmax) for a 2-D float32 CUDA tensor: one device pass (fs_row_absmax) that both
    validates finiteness and returns max_j |t[i, j]| per row (float32, device) — the exact F16X2
    row scales for every later solve on these scores."""
    import torch
    if t.dim() != 2 or t.stride(1) != 1 or t.dtype not in (torch.float32, torch.float64):
        raise ValueError("row_absmax needs a 2-D float tensor with unit column stride")
    out = torch.empty(t.shape[0], dtype=torch.float32, device=t.device)
    lib = load()
    with torch.cuda.device(t.device):
        rc = lib.fs_row_absmax(FS_F64 if t.dtype == torch.float64 else FS_F32, t.data_ptr(), t.shape[0], t.shape[1],
                               t.stride(0), out.data_ptr(), torch.cuda.current_stream(t.device).cuda_stream)
    if rc not in (0, 1):
        raise NativeLibraryError(f"fs_row_absmax failed (status {rc})")
    return rc == 0, out


def context_for(device: int, n: int, m: int) -> Context:
    """Return a cached context on `device` large enough for (n, m).

    A context that must grow keeps the old bounds only while that costs little: the tiled score
    copy is sized n_max * m_max, so (8192, 1e6) followed by (1024, 3e6) must become a (1024, 3e6)
    context, not an (8192, 3e6) one (98 GB)."""
    ctx = _contexts.get(device)
    if ctx is None or ctx.n_max < n or ctx.m_max < m:
        n_max = max(n, ctx.n_max if ctx else 0)
        m_max = max(m, ctx.m_max if ctx else 0)
        if n_max * m_max > 2 * n * m:
            n_max, m_max = n, m
        if ctx is not None:
            ctx.close()
        ctx = Context(device, n_max, m_max)
        _contexts[device] = ctx
    return ctx


def release_contexts():
    for ctx in list(_contexts.values()):
        ctx.close()
    _contexts.clear()
