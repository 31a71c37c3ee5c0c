"""GPU parity of the code paths that environment switches select (each case runs in a fresh
process, because the switches are read once per process):

  FS_TILE_CAP_MB  caps the tiled copy of S -> the K-chunked Gram (retile a column range, SYRK its
                  K-blocks, accumulate), the path that lets n = 16384, m = 2e6 fit on one B200
  FS_F16_RING=1   the F16X2 ring SYRK (each tile split once into an L2-resident ring)
  FS_TRSV_FLAGS=0 the single-CTA TRSV pair instead of the flag-chained one
  FS_DZ_ASYNC=0   the refinement's convergence test through a stream sync instead of a side stream
  FS_POTRF_CLUSTER_BWD=0  potrf's own backward solve instead of the TRSV cluster's backward half

Tolerances: fp32 modes relerr(x) <= 1e-6 vs the reference's fp64 solve of the same
fp32-rounded system; the chunked Gram vs the one-shot Gram <= 2e-6 of max |G| (the same split
products, but each chunk's split-K plan groups the tensor core's fp32 accumulation differently).
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import fisher_oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASE = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2310_17556_b200 as fsb
from oracle import fisher_oracle as O
n, m, prec, entry, refine = {n}, {m}, {prec!r}, {entry!r}, {refine!r}
S, v, lam = O.generate_problem(7, n, m, 1e-3)
S32, v32 = S.astype(np.float32), v.astype(np.float32)
if entry == "device":
    sm = fsb.ScoreMatrix(torch.from_numpy(S32).cuda())
    system = fsb.DampedSystem(sm, lam, torch.from_numpy(v32).cuda())
    G = fsb.gram_packed(sm, lam, precision=prec).cpu().numpy()
else:
    system = fsb.DampedSystem(fsb.ScoreMatrix(S32, defer=True), lam, v32)
    G = np.zeros(1)
sol = fsb.solve_chol(system, precision=prec, refine=refine)
x = sol.x.cpu().numpy() if hasattr(sol.x, "cpu") else np.asarray(sol.x)
np.savez({out!r}, x=x, G=G)
print(json.dumps({{"rel_residual": float(sol.rel_residual)}}))
'''


def run_case(tmp_path, env, n, m, prec, entry="device", refine=0):
    out = str(tmp_path / f"case_{abs(hash((tuple(sorted(env.items())), n, m, prec, entry)))}.npz")
    code = CASE.format(root=ROOT, n=n, m=m, prec=prec, entry=entry, refine=refine, out=out)
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    info = json.loads(r.stdout.strip().splitlines()[-1])
    d = np.load(out)
    return d["x"], d["G"], info


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")


def reference(n, m):
    S, v, lam = O.generate_problem(7, n, m, 1e-3)
    S64, v64 = S.astype(np.float32).astype(np.float64), v.astype(np.float32).astype(np.float64)
    return O.solve_chol(S64, v64, lam)


@pytest.mark.parametrize("prec", ["f16x2", "tf32x3"])
@pytest.mark.parametrize("n,m", [(300, 70001), (1024, 50000)])
def test_k_chunked_gram_matches_one_shot_and_oracle(gpu, tmp_path, prec, n, m):
    # a 6 MB cap: the planes of (n, m) need ~n m 4 bytes, so the Gram runs in many K-chunks
    x1, G1, _ = run_case(tmp_path, {}, n, m, prec)
    x2, G2, _ = run_case(tmp_path, {"FS_TILE_CAP_MB": "6"}, n, m, prec)
    assert np.abs(G2 - G1).max() <= 2e-6 * np.abs(G1).max()
    ref = reference(n, m)
    assert O.rel_err(x2, ref.x) <= 1e-6
    assert O.rel_err(x1, ref.x) <= 1e-6


@pytest.mark.parametrize("prec", ["f16x2", "tf32x3"])
def test_k_chunked_host_entry(gpu, tmp_path, prec):
    n, m = 512, 90001
    # planes of all of S: 184 MB > the 64 MB cap; the host entry's ~32 MB upload chunks fit
    x, _, info = run_case(tmp_path, {"FS_TILE_CAP_MB": "64"}, n, m, prec, entry="host")
    assert O.rel_err(x, reference(n, m).x) <= 1e-6


@pytest.mark.parametrize("n,m", [(128, 70000), (300, 65573), (1024, 100000), (2048, 40000)])
def test_ring_syrk_gram_is_bit_identical_and_solves(gpu, tmp_path, n, m):
    x1, G1, _ = run_case(tmp_path, {"FS_F16_RING": "0"}, n, m, "f16x2")
    x2, G2, _ = run_case(tmp_path, {"FS_F16_RING": "1"}, n, m, "f16x2")
    assert np.array_equal(G1, G2)          # same tiles, same MMA order: bit-identical Gram
    assert O.rel_err(x2, reference(n, m).x) <= 1e-6


def test_refinement_step_decisions_sync_or_side_stream_bit_identical(gpu, tmp_path):
    """The z-space steps' convergence numbers come back on a side stream while the x + y pass runs
    (default) or through a stream sync (FS_DZ_ASYNC=0): the same decisions, the same bits."""
    n, m = 1024, 200000
    x1, _, i1 = run_case(tmp_path, {}, n, m, "f16x2", refine=4)
    x2, _, i2 = run_case(tmp_path, {"FS_DZ_ASYNC": "0"}, n, m, "f16x2", refine=4)
    assert np.array_equal(x1, x2) and i1["rel_residual"] == i2["rel_residual"] <= 1e-10


@pytest.mark.parametrize("n", [130, 700, 1024, 1100])
def test_potrf_backward_on_the_trsv_cluster(gpu, tmp_path, n):
    """n <= 1024: potrf's fused backward solve runs as the TRSV cluster's backward half
    (FS_POTRF_CLUSTER_BWD=0: inside the persistent kernel); n = 1100 keeps the in-kernel solve.
    The same z up to rounding order: x to the fp64 solve's 1e-10 either way."""
    m = 40000
    ref = reference(n, m)
    for env in ({}, {"FS_POTRF_CLUSTER_BWD": "0"}):
        x, _, info = run_case(tmp_path, env, n, m, "f16x2", refine=2)
        assert O.rel_err(x, ref.x) <= 1e-10, (env, O.rel_err(x, ref.x))
        assert info["rel_residual"] <= 1e-10


@pytest.mark.parametrize("n", [130, 1000])
def test_trsv_pair_variants_agree(gpu, tmp_path, n):
    """single-CTA, flag-chained multi-CTA and cluster (DSMEM) TRSV pairs in the refinement steps:
    the same z up to rounding order (x to the fp64 solve's 1e-10)."""
    m = 60000
    ref = reference(n, m)
    for env in ({"FS_TRSV_FLAGS": "0"}, {"FS_TRSV_CLUSTER": "0"}, {}):
        x, _, info = run_case(tmp_path, env, n, m, "f16x2", refine=2)
        assert O.rel_err(x, ref.x) <= 1e-10, (env, O.rel_err(x, ref.x))
        assert info["rel_residual"] <= 1e-10


POTRF_CASE = r'''
import sys, json, numpy as np
sys.path.insert(0, {root!r})
import paper_2310_17556_b200 as fsb
from paper_2310_17556_b200.solvers import _cholesky_lower
from oracle import fisher_oracle as O
n, bad = {n}, {bad}
rng = np.random.Generator(np.random.PCG64(n + 7))
A = rng.standard_normal((n, n + 64))
W = A @ A.T / n + 0.1 * np.eye(n)
if bad >= 0:
    W[bad, :bad] = W[bad - 1, :bad]
    W[:bad, bad] = W[bad, :bad]
    W[bad, bad] = W[bad - 1, bad - 1] - 1.0
    try:
        O.cholesky_lower(W)
        ref_piv = None
    except O.OracleFactorizationError as e:
        ref_piv = e.pivot
    try:
        _cholesky_lower(W)
        piv = None
    except fsb.FactorizationError as e:
        piv = e.pivot
    print(json.dumps({{"piv": piv, "ref_piv": ref_piv}}))
else:
    L = _cholesky_lower(W)
    ref = O.cholesky_lower(W)
    print(json.dumps({{"err": float(np.abs(L - ref).max() / np.abs(ref).max()),
                      "upper_zero": bool(np.array_equal(np.triu(L, 1), np.zeros((n, n))))}}))
'''


def run_potrf(env, n, bad=-1):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", POTRF_CASE.format(root=ROOT, n=n, bad=bad)], env=e, capture_output=True,
                       text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("n,minn", [(700, "300"), (1100, "300"), (4500, "4096"), (6145, "6144")])
def test_blocked_potrf_matches_lapack(gpu, n, minn):
    """256-wide block columns: diagonal blocks by the persistent kernel, GEMM-form panel TRSM, DMMA
    trailing tiles (FS_POTRF_BLOCKED_MINN lowers the size where it takes over)."""
    info = run_potrf({"FS_POTRF_BLOCKED_MINN": minn}, n)
    assert info["err"] <= 1e-10 and info["upper_zero"], info


@pytest.mark.parametrize("n,bad", [(700, 5), (700, 300), (700, 699), (1100, 513)])
def test_blocked_potrf_pivot_index(gpu, n, bad):
    info = run_potrf({"FS_POTRF_BLOCKED_MINN": "300"}, n, bad)
    assert info["ref_piv"] == bad and info["piv"] == bad, info


def test_repeated_solves_are_bit_identical(gpu):
    """Race check by repetition (compute-sanitizer is closed on this pool): every cross-CTA protocol
    on the path — the SYRK's CTA-pair barriers, the split-K reduce, the persistent potrf's grid
    barriers and flags, the cluster TRSV's DSMEM pushes, the x + y pass's exchange, the block
    Jacobi's phases — runs in a fixed order, so repeated solves must agree bit for bit."""
    import paper_2310_17556_b200 as fsb
    S, v, lam = O.generate_problem(99, 1000, 60000, 1e-3)
    S32, v32 = S.astype(np.float32), v.astype(np.float32)
    dev = torch.device("cuda", 0)
    system = fsb.DampedSystem(fsb.ScoreMatrix(torch.from_numpy(S32).to(dev)), lam, torch.from_numpy(v32).to(dev))
    for fn, kw in ((fsb.solve_chol, {}), (fsb.solve_chol, {"precision": "fp64"}), (fsb.solve_svd_eigh, {})):
        ref = fn(system, **kw)
        x0 = ref.x.cpu().numpy()
        for _ in range(6):
            sol = fn(system, **kw)
            assert np.array_equal(sol.x.cpu().numpy(), x0), (fn.__name__, kw)
            assert sol.rel_residual == ref.rel_residual
