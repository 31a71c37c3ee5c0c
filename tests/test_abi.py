"""The C-ABI library loads and exports every symbol include/fs.h declares (CPU only:
no compute calls without a GPU)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "fs.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(fs_[a-z0-9_]+)\s*\(", text))
    names.discard("fs_allreduce_fn")
    return sorted(names)


def test_header_declares_the_solver_surface():
    names = declared_symbols()
    for required in ("fs_chol_solve", "fs_gram_packed", "fs_potrf", "fs_trsv_pair", "fs_gemv_rows",
                     "fs_gemv_cols_solve", "fs_residual_cols", "fs_ctx_create", "fs_ctx_destroy"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2310_17556_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2310_17556_b200.build import build
        build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), f"{name} declared in fs.h but not exported"


def test_ctypes_signatures_cover_the_header():
    from paper_2310_17556_b200 import _lib
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_version_and_workspace_query_without_gpu():
    from paper_2310_17556_b200 import _lib
    lib = _lib.load()
    assert lib.fs_version().decode().startswith("fisher-b200")
    small = lib.fs_workspace_bytes(64, 4096, _lib.FS_F64, _lib.FS_PREC_FP64)
    big = lib.fs_workspace_bytes(1024, 1000000, _lib.FS_F32, _lib.FS_PREC_TF32X3)
    assert 0 < small < big
    # workspace is O(n^2 + n m / chunk + m): far below the n*m*8 bytes of S itself
    assert big < 1024 * 1000000 * 8


def test_missing_library_fails_loudly(tmp_path):
    from paper_2310_17556_b200 import _lib
    with pytest.raises(_lib.NativeLibraryError):
        saved = _lib._lib
        _lib._lib = None
        try:
            _lib.load(str(tmp_path / "nope.so"))
        finally:
            _lib._lib = saved


def test_no_oracle_import_in_product():
    pkg = os.path.join(ROOT, "paper_2310_17556_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), f


def test_context_growth_does_not_multiply_bounds(monkeypatch):
    """context_for keeps old bounds only when cheap: (8192, 1e6) then (1024, 3e6) must not become
    an (8192, 3e6) workspace (the sweep that found it ran out of HBM)."""
    from paper_2310_17556_b200 import _lib

    class FakeCtx:
        def __init__(self, device, n_max, m_max):
            self.device, self.n_max, self.m_max = device, n_max, m_max

        def close(self):
            pass

    monkeypatch.setattr(_lib, "Context", FakeCtx)
    monkeypatch.setattr(_lib, "_contexts", {})
    c = _lib.context_for(0, 8192, 1_000_000)
    assert (c.n_max, c.m_max) == (8192, 1_000_000)
    c = _lib.context_for(0, 1024, 3_000_000)
    assert (c.n_max, c.m_max) == (1024, 3_000_000)
    c = _lib.context_for(0, 2048, 3_000_000)          # 2x the area of the request: keep growing
    assert (c.n_max, c.m_max) == (2048, 3_000_000)
    assert _lib.context_for(0, 1024, 2_000_000) is c  # fits: reused
