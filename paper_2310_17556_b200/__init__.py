"""paper_2310_17556_b200 — B200-native drop-in for fisher_solve's Cholesky hot path.

Solves (S^T S + lam I) x = v for wide score matrices (m >> n) by the paper's
Algorithm 1 with hand-written sm_100a kernels behind the C ABI of include/fs.h:
tcgen05/TMEM split-precision (or exact fp64) Gram, fp64 blocked Cholesky, TRSV pair, and
HBM-streaming GEMVs with a fused (v - S^T z)/lam epilogue; the eigh / direct-SVD comparison
routes and the complex variants on the same kernels.  Multi-GPU: the m axis
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
    as_scores,
    as_system,
    gram,
    gram_packed,
    residual,
)
from .fmat import FmatError, read_matrix, read_vector, write_matrix, write_vector
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
    resolve_solver,
    solve_svd_direct,
    solve_svd_eigh,
    solve_svd_from_factors,
    ThinSvd,
    eigh_gram,
    thin_svd_direct,
    thin_svd_eigh,
)

__version__ = "0.1.0"
