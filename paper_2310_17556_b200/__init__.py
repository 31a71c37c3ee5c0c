"""paper_2310_17556_b200 — B200-native drop-in for fisher_solve's Cholesky hot path.

Solves (S^T S + lam I) x = v for wide score matrices (m >> n) by the paper's
Algorithm 1 with hand-written sm_100a kernels behind the C ABI of include/fs.h:
tcgen05/TMEM 3xTF32 (or exact fp64) Gram, fp64 blocked Cholesky, TRSV pair, and
HBM-streaming GEMVs with a fused (v - S^T z)/lam epilogue.  Multi-GPU: the m axis
is column-sharded with one NCCL all-reduce of [W | u] (see distributed.py).

The public names mirror /root/reference/pkg/src/fisher_solve/__init__.py for the
solver path.  There is no CPU fallback: the product raises if libfisher_b200.so
or a CUDA device is missing.
"""

from .core import (
    EPS,
    DampedSystem,
    FactorizationError,
    Method,
    ScalarKind,
    ScoreMatrix,
    Solution,
    Variant,
    WorkspaceMeter,
    gram,
    gram_packed,
    residual,
)
from .solvers import (
    DEFAULT_NAIVE_CAP,
    DEFAULT_SIGMA_FLOOR,
    REFINE_ABOVE_REL,
    CholWorkspace,
    cholesky_lower_device,
    fp32_residual_bound,
    solve_chol,
    solve_chol_hermitian,
    solve_realpart,
    solve_svd_direct,
    solve_svd_eigh,
    ThinSvd,
    eigh_gram,
    thin_svd_eigh,
)

__version__ = "0.1.0"
