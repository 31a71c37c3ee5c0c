"""The product's multi-rank path at world size 2-3 on one GPU.

Every rank is its own process on cuda:0 and calls sharded_solve_chol_fused -> ONE fs_chol_solve
(or fs_chol_solve_host) with the C ABI's all-reduce callback over a gloo process group (NCCL
cannot put two ranks on one device; gloo all-reduces the CUDA buffers through the host).  The
ranks' kernels never wait on one another — the exchanges are host-side — so this exercises the
fused path's collective protocol exactly as an 8-GPU NCCL job would, minus the transport.

Checked against the CPU oracle (f16x2: relerr <= 1e-6, fp64: <= 1e-10), plus the failure
protocol: refinement steps, an F16X2 overflow on one rank only (every rank retries in TF32X3),
a non-PD Gram (FactorizationError on every rank), a non-finite shard on one rank (ValueError on
every rank, no hang), and a zero-column shard (m < world).
"""

import multiprocessing as mp
import os
import socket
import traceback

import numpy as np
import pytest
import torch

from oracle import fisher_oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case_system(case):
    """(S, v, lam, precision, refine, mutate) for one scenario; identical in every process."""
    if case == "zero_col":
        S, v, lam = O.generate_problem(71, 16, 2, 1e-2)
        return S.astype(np.float32), v.astype(np.float32), lam, "f16x2", 0
    S, v, lam = O.generate_problem(70, 96, 12000, 1e-3)
    S32, v32 = S.astype(np.float32), v.astype(np.float32)
    if case == "fp64":
        return S, v, lam, "fp64", 1
    if case == "not_pd":
        # two finite rows whose products overflow: G_00 = +inf (accepted, > 0), G_10 = +-inf or NaN,
        # so the updated pivot 1 is NaN on every rank -> FactorizationError(pivot=1) everywhere
        S = np.array(S)
        S[:2] *= 1e200
        return S, v, 1.0, "fp64", 0
    if case == "overflow_one_rank":
        S32 = np.array(S32)
        # rank 1's shard starts at column 6000: its first 4096 columns (the sampled scale) tiny for
        # row 5, a huge entry past the sample -> fp16 overflow on rank 1 only
        S32[5, 6000:10200] *= np.float32(1e-6)
        S32[5, 11000] = np.float32(60.0)
        return S32, v32, 1e-2, "f16x2", 0
    return S32, v32, lam, "f16x2", (4 if case == "refine" else 0)


def _worker(rank, world, port, case, entry, q):
    try:
        import sys
        sys.path.insert(0, ROOT)
        import datetime
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=90))
        import paper_2310_17556_b200 as fsb
        from paper_2310_17556_b200.distributed import column_shard, sharded_solve_chol_fused
        S, v, lam, prec, refine = _case_system(case)
        a, b = column_shard(S.shape[1], world, rank)
        Sk, vk = np.ascontiguousarray(S[:, a:b]), np.ascontiguousarray(v[a:b])
        if case == "nonfinite_one_rank" and rank == world - 1:
            Sk[3, 7] = np.nan
        try:
            if entry == "host":
                sol = sharded_solve_chol_fused(Sk, vk, lam, precision=prec, refine=refine)
                x = np.asarray(sol.x_local).copy()
            else:
                sol = sharded_solve_chol_fused(torch.from_numpy(Sk).cuda(), torch.from_numpy(vk).cuda(), lam,
                                               precision=prec, refine=refine)
                x = sol.x_local.cpu().numpy()
            q.put((rank, "ok", (a, b, x, sol.rel_residual)))
        except fsb.FactorizationError as e:
            q.put((rank, "FactorizationError", e.pivot))
        except ValueError as e:
            q.put((rank, "ValueError", str(e)))
        dist.destroy_process_group()
    except Exception:
        q.put((rank, "crash", traceback.format_exc()))


def run_world(world, case, entry, timeout=240):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, entry, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(world):
            r, kind, payload = q.get(timeout=timeout)
            out[r] = (kind, payload)
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    crashes = [v[1] for v in out.values() if v[0] == "crash"]
    assert not crashes, crashes[0]
    assert len(out) == world, f"ranks {sorted(set(range(world)) - set(out))} did not finish (hang)"
    return out


def _assemble(out, m):
    x = np.empty(m)
    rels = set()
    for kind, (a, b, xk, rel) in out.values():
        assert kind == "ok"
        x[a:b] = xk
        rels.add(rel)
    assert len(rels) == 1          # every rank reports the same (all-reduced) residual
    return x, rels.pop()


@pytest.fixture(scope="module", autouse=True)
def gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("entry", ["device", "host"])
def test_sharded_fused_matches_oracle(world, entry):
    S, v, lam, prec, refine = _case_system("plain")
    out = run_world(world, "plain", entry)
    x, rel = _assemble(out, S.shape[1])
    ref = O.solve_chol(S.astype(np.float64), v.astype(np.float64), lam)
    assert O.rel_err(x, ref.x) <= 1e-6, O.rel_err(x, ref.x)
    assert rel <= 4 * 2.0 ** -24 * 200.0 / lam


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fused_fp64_and_refinement(world):
    S, v, lam, _, _ = _case_system("fp64")
    out = run_world(world, "fp64", "device")
    x, rel = _assemble(out, S.shape[1])
    ref = O.solve_chol(S, v, lam)
    assert O.rel_err(x, ref.x) <= 1e-10
    assert rel <= 1e-8
    S, v, lam, _, _ = _case_system("refine")
    out = run_world(world, "refine", "device")
    x, rel4 = _assemble(out, S.shape[1])
    ref = O.solve_chol(S.astype(np.float64), v.astype(np.float64), lam)
    assert O.rel_err(x, ref.x) <= 1e-7
    out0 = run_world(world, "plain", "device")
    _, rel0 = _assemble(out0, S.shape[1])
    assert rel4 < 0.2 * rel0, (rel4, rel0)          # the correction steps contracted collectively


@pytest.mark.parametrize("entry", ["device", "host"])
def test_sharded_overflow_on_one_rank_retries_everywhere(entry):
    S, v, lam, _, _ = _case_system("overflow_one_rank")
    out = run_world(2, "overflow_one_rank", entry)
    x, _ = _assemble(out, S.shape[1])
    ref = O.solve_chol(S.astype(np.float64), v.astype(np.float64), lam)
    assert O.rel_err(x, ref.x) <= 1e-6


def test_sharded_not_pd_raises_on_every_rank():
    out = run_world(3, "not_pd", "device")
    assert all(kind == "FactorizationError" for kind, _ in out.values()), out
    assert {p for _, p in out.values()} == {1}


@pytest.mark.parametrize("entry", ["device", "host"])
def test_sharded_nonfinite_shard_fails_every_rank_without_hang(entry):
    out = run_world(3, "nonfinite_one_rank", entry)
    assert all(kind == "ValueError" for kind, _ in out.values()), out
    assert "finite" in out[2][1]
    assert "peer" in out[0][1] and "peer" in out[1][1]


def test_sharded_zero_column_shard():
    """m = 2 over 3 ranks: rank 0's shard is empty (column_shard gives [0, 0))."""
    S, v, lam, _, _ = _case_system("zero_col")
    out = run_world(3, "zero_col", "device")
    x, _ = _assemble(out, S.shape[1])
    ref = O.solve_chol(S.astype(np.float64), v.astype(np.float64), lam)
    assert O.rel_err(x, ref.x) <= 1e-6
