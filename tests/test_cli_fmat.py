"""FMAT interchange and the GPU command line tool (fmat.py, cli.py of the reference)."""

import os

import numpy as np
import pytest

from oracle import fisher_oracle as O
from paper_2310_17556_b200 import fmat
from paper_2310_17556_b200.cli import build_parser, generate_problem, run_cli


def test_fmat_round_trip_is_bit_exact(tmp_path):
    rng = np.random.Generator(np.random.PCG64(3))
    a = rng.standard_normal((7, 11))
    c = a + 1j * rng.standard_normal((7, 11))
    for arr in (a, c, np.arange(6).reshape(2, 3)):
        p = tmp_path / "m.fmat"
        fmat.write_matrix(p, arr)
        b = fmat.read_matrix(p, pinned=False)
        assert b.dtype == (np.complex128 if np.iscomplexobj(arr) else np.float64)
        assert np.array_equal(b, arr) and b.tobytes() == np.asarray(arr, b.dtype).tobytes()
    fmat.write_vector(tmp_path / "v.fmat", a[0])
    assert np.array_equal(fmat.read_vector(tmp_path / "v.fmat"), a[0])


def test_fmat_rejects_malformed_files(tmp_path):
    p = tmp_path / "bad.fmat"
    fmat.write_matrix(p, np.ones((2, 2)))
    blob = p.read_bytes()
    for bad in (b"XMAT" + blob[4:], blob[:4] + b"\x02" + blob[5:], blob[:5] + b"\x07" + blob[6:], blob[:-8], blob[:10]):
        p.write_bytes(bad)
        with pytest.raises(fmat.FmatError):
            fmat.read_matrix(p, pinned=False)
    with pytest.raises(fmat.FmatError):
        fmat.write_matrix(tmp_path / "x.fmat", np.ones(3))
    p.write_bytes(blob)
    with pytest.raises(fmat.FmatError):
        fmat.read_vector(p)


@pytest.mark.parametrize("kind", ["real", "complex", "structured"])
def test_cli_generator_matches_the_pinned_oracle(kind):
    """The CLI's generator reproduces bench.py:127-171's stream (the oracle's restatement is pinned
    to the reference's own generator by tests/test_oracle_golden.py)."""
    S, v, lam, f = generate_problem(5, 9, 40, 1e-3, kind)
    if kind == "real":
        So, vo, _ = O.generate_problem(5, 9, 40, 1e-3)
        assert np.array_equal(S, So) and np.array_equal(v, vo)
    elif kind == "complex":
        So, vo, _ = O.generate_problem_complex(5, 9, 40, 1e-3)
        assert np.array_equal(S, So) and np.array_equal(v, vo)
    else:
        So, _, _ = O.generate_problem(5, 9, 40, 1e-3)
        assert np.array_equal(S, So) and f is not None and np.allclose(v, f @ S, rtol=0, atol=0)


def test_cli_gen_and_argument_errors(tmp_path, capsys):
    prefix = str(tmp_path / "p")
    assert run_cli(["gen", "--n", "4", "--m", "12", "--seed", "2", "--out", prefix]) == 0
    S = fmat.read_matrix(prefix + ".S.fmat", pinned=False)
    So, vo, _ = O.generate_problem(2, 4, 12, 1e-3)
    assert np.array_equal(S, So)
    assert np.array_equal(fmat.read_vector(prefix + ".v.fmat"), vo)
    assert run_cli(["solve", prefix + ".S.fmat", prefix + ".v.fmat", "--method", "cg"]) == 2      # not provided
    assert run_cli(["gen", "--n", "0", "--m", "3", "--out", prefix]) == 1
    assert build_parser().parse_args(["scaling", "--method", "chol", "--fix", "n=8", "--vary", "m=16:64:3"]).vary[1]


@pytest.mark.gpu
def test_cli_solve_check_bench_on_gpu(tmp_path, capsys):
    prefix = str(tmp_path / "q")
    assert run_cli(["gen", "--n", "32", "--m", "500", "--seed", "4", "--lambda", "0.01", "--out", prefix]) == 0
    out = str(tmp_path / "x.fmat")
    assert run_cli(["solve", prefix + ".S.fmat", prefix + ".v.fmat", "--method", "chol", "--lambda", "0.01",
                    "--out", out]) == 0
    S, v, lam = O.generate_problem(4, 32, 500, 0.01)
    assert O.rel_err(fmat.read_vector(out), O.solve_chol(S, v, lam).x) <= 1e-10
    for method in ("eigh", "svd"):
        assert run_cli(["solve", prefix + ".S.fmat", prefix + ".v.fmat", "--method", method, "--lambda", "0.01",
                        "--out", out]) == 0
        assert O.rel_err(fmat.read_vector(out), O.solve_chol(S, v, lam).x) <= 1e-8
    assert run_cli(["check", "--n", "24", "--m", "300", "--lambda", "0.01"]) == 0
    assert "all checks passed" in capsys.readouterr().out
    assert run_cli(["bench", "--n", "64", "--m", "4096", "--method", "chol", "--repeats", "2", "--warmup", "1"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "method,n,m,lambda,seed,repeats,median_s,min_s,rel_residual,status"
    assert lines[1].startswith("chol,64,4096,") and lines[1].endswith(",ok")
