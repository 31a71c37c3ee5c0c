"""The bench's own code paths on the GPU at a small shape: the N=1 line, the multi-GPU path on a
one-rank NCCL group (--sharded: one fs_chol_solve per rank with the all-reduce callback, as the
driver's torchrun N>1 runs use it) and the reference arm — so the driver's round-end bench and
scaling runs cannot hit an untested branch.  Each JSON line must carry the contract's keys."""

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "clocks"}


def run_bench(*extra, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, "bench.py", *extra], cwd=ROOT, env=e, capture_output=True, text=True,
                       timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert lines, r.stdout[-2000:]
    return json.loads(lines[-1])


@pytest.fixture(scope="module")
def gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")


SMALL = ("--n", "256", "--m", "200000", "--steps", "3", "--warmup", "3", "--e2e-steps", "2", "--no-pageable")


def test_bench_line_single_gpu(gpu):
    d = run_bench(*SMALL, "--no-cpu-baseline")
    assert KEYS <= set(d) and d["n_gpus"] == 1 and d["value"] > 0
    assert d["roofline"]["bound"] == "tensor" and d["gpu_launches"] > 0
    assert d["rel_residual"] <= 1e-8
    assert d["e2e"]["h2d_bytes_per_step"] > 0


def test_bench_sharded_one_rank_nccl(gpu):
    env = {"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": "29561", "RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0"}
    d = run_bench(*SMALL, "--sharded", "--philox", "--no-cpu-baseline", env=env)
    assert KEYS <= set(d) and d["value"] > 0 and d["rel_residual"] <= 1e-8


def test_bench_reference_arm(gpu):
    d = run_bench("--impl", "reference", "--n", "64", "--m", "4096", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
