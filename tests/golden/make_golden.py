"""Generate golden fixtures by running the REAL reference package.

Run in the survey/build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``fisher_solve`` from /root/reference/pkg/src, evaluates the
reference's own entry points (solve_chol, gram, _cholesky_lower,
solve_svd_eigh, solve_svd_direct, generate_problem) on seeded inputs and
writes ``tests/golden/golden.npz`` plus ``tests/golden/MANIFEST.json``.
Inputs are NOT stored when they can be regenerated from a PCG64 seed; a
checksum of each regenerated S is stored instead so tests can prove the
generator restatement matches.  Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

import fisher_solve as fs  # noqa: E402
from fisher_solve.solvers import _cholesky_lower  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def checksum(a: np.ndarray) -> list:
    a = np.asarray(a, dtype=np.float64)
    return [float(a.sum()), float(np.abs(a).sum()), float(a.ravel()[0]), float(a.ravel()[-1])]


def main():
    out = {}
    manifest = {"reference": "fisher_solve " + fs.__version__, "numpy": np.__version__, "cases": {}}

    # --- hand KATs (tests/test_solvers.py:82-107, test_core.py:97-108) -----------------
    kat = fs.solve_chol(fs.DampedSystem(fs.ScoreMatrix([[1.0, 2.0]]), 1.0, [1.0, 1.0]))
    out["kat_hand_x"] = kat.x
    z = fs.solve_chol(fs.DampedSystem(fs.ScoreMatrix(np.zeros((3, 5))), 2.0,
                                      [2.0, 4.0, 6.0, 8.0, 10.0]))
    out["kat_zero_scores_x"] = z.x
    try:
        _cholesky_lower(np.array([[1.0, 2.0], [2.0, 1.0]]))
        raise SystemExit("expected FactorizationError")
    except fs.FactorizationError as e:
        out["kat_potrf_pivot"] = np.array([e.pivot])

    # --- seeded random systems through the reference's own generators -----------------
    # (name, generator, seed, n, m, lam)
    cases = [
        ("rs_42_8_50", "random_system", 42, 8, 50, 1e-3),
        ("gp_0_64_4096", "generate_problem", 0, 64, 4096, 1e-3),       # BASELINE configs[0]
        ("gp_1_100_1000", "generate_problem", 1, 100, 1000, 1e-3),
        ("gp_2_129_3001", "generate_problem", 2, 129, 3001, 1e-2),
        ("gp_3_1_7", "generate_problem", 3, 1, 7, 1.0),
        ("gp_4_16_64", "generate_problem", 4, 16, 64, 1e-6),
        ("gp_5_200_20000", "generate_problem", 5, 200, 20000, 1e-3),
        ("gp_6_40_600", "generate_problem", 6, 40, 600, 1e-5),       # triggers refinement
    ]
    for name, gen, seed, n, m, lam in cases:
        if gen == "random_system":
            rng = np.random.Generator(np.random.PCG64(seed))
            S = fs.ScoreMatrix(rng.standard_normal((n, m)) / np.sqrt(n))
            system = fs.DampedSystem(S, lam, rng.standard_normal(m))
        else:
            system = fs.generate_problem(seed, n, m, lam).system
        A = system.S.data
        sol = fs.solve_chol(system)
        W = fs.gram(system.S, lam)
        L = _cholesky_lower(W)
        out[f"{name}_x"] = sol.x
        out[f"{name}_res"] = np.array([sol.abs_residual, sol.rel_residual])
        out[f"{name}_u"] = A @ system.v
        if n <= 256:
            out[f"{name}_W"] = W
            out[f"{name}_L"] = L
        if m <= 4096:
            out[f"{name}_eigh_x"] = fs.solve_svd_eigh(system).x
            out[f"{name}_svd_x"] = fs.solve_svd_direct(system).x
        manifest["cases"][name] = {"gen": gen, "seed": seed, "n": n, "m": m, "lam": lam,
                                   "S_checksum": checksum(A), "v_checksum": checksum(system.v),
                                   "rel_residual": sol.rel_residual}

    # --- fp32-rounded systems: the identical system the fp32 GPU modes solve ----------
    f32_cases = [("f32_0_64_4096", 0, 64, 4096, 1e-3), ("f32_7_256_32768", 7, 256, 32768, 1e-3),
                 ("f32_8_300_10000", 8, 300, 10000, 1e-2)]
    for name, seed, n, m, lam in f32_cases:
        p = fs.generate_problem(seed, n, m, lam).system
        S32 = p.S.data.astype(np.float32).astype(np.float64)
        v32 = p.v.astype(np.float32).astype(np.float64)
        system = fs.DampedSystem(fs.ScoreMatrix(S32), lam, v32)
        sol = fs.solve_chol(system)
        out[f"{name}_x"] = sol.x
        out[f"{name}_res"] = np.array([sol.abs_residual, sol.rel_residual])
        manifest["cases"][name] = {"gen": "generate_problem+f32", "seed": seed, "n": n, "m": m,
                                   "lam": lam, "S_checksum": checksum(S32),
                                   "rel_residual": sol.rel_residual}

    # --- complex scores (Kind.COMPLEX_GAUSSIAN): Hermitian and real-part variants ---------
    cx_cases = [("cx_10_16_200", 10, 16, 200, 1e-3), ("cx_11_64_2048", 11, 64, 2048, 1e-2)]
    for name, seed, n, m, lam in cx_cases:
        system = fs.generate_problem(seed, n, m, lam, "complex").system
        sol = fs.solve_chol_hermitian(system)
        out[f"{name}_herm_x"] = sol.x
        out[f"{name}_herm_res"] = np.array([sol.abs_residual, sol.rel_residual])
        rp = fs.DampedSystem(system.S, lam, system.v.real.copy())
        solr = fs.solve_realpart(rp)
        out[f"{name}_real_x"] = solr.x
        out[f"{name}_real_res"] = np.array([solr.abs_residual, solr.rel_residual])
        manifest["cases"][name] = {"gen": "generate_problem+complex", "seed": seed, "n": n, "m": m, "lam": lam,
                                   "S_checksum": checksum(system.S.data.real) + checksum(system.S.data.imag),
                                   "rel_residual": sol.rel_residual}

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
