"""Pin the CPU oracle (oracle/fisher_oracle.py) against fixtures produced by the REAL
reference package (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import fisher_oracle as O

from conftest import regenerate


def test_generator_restatement_matches_reference(manifest):
    for name, case in manifest["cases"].items():
        S, v, lam = regenerate(case)
        cs = case["S_checksum"]
        assert S.shape == (case["n"], case["m"])
        parts = [S.real, S.imag] if np.iscomplexobj(S) else [S]
        for k, P in enumerate(parts):
            c = cs[4 * k: 4 * k + 4]
            assert float(P.ravel()[0]) == c[2] and float(P.ravel()[-1]) == c[3], name
            assert abs(float(P.sum()) - c[0]) <= 1e-9 * max(1.0, abs(c[1])), name


@pytest.mark.parametrize("name", ["cx_10_16_200", "cx_11_64_2048"])
def test_complex_variants_match_reference(name, golden, manifest):
    """Oracle restatements of solve_chol_hermitian and solve_realpart vs the real reference."""
    S, v, lam = regenerate(manifest["cases"][name])
    h = O.solve_chol_hermitian(S, v, lam)
    assert O.rel_err(h.x, golden[f"{name}_herm_x"]) <= 1e-12
    assert abs(h.rel_residual - golden[f"{name}_herm_res"][1]) <= 1e-3 * golden[f"{name}_herm_res"][1] + 1e-18
    r = O.solve_realpart(S, v.real.copy(), lam)
    assert O.rel_err(r.x, golden[f"{name}_real_x"]) <= 1e-12
    assert abs(r.rel_residual - golden[f"{name}_real_res"][1]) <= 1e-3 * golden[f"{name}_real_res"][1] + 1e-18


def test_hand_kats(golden):
    # tests/test_solvers.py:82-91 (hand example and exact zero-score case)
    sol = O.solve_chol(np.array([[1.0, 2.0]]), np.array([1.0, 1.0]), 1.0)
    np.testing.assert_allclose(sol.x, golden["kat_hand_x"], atol=1e-14)
    np.testing.assert_allclose(sol.x, [0.5, 0.0], atol=1e-14)
    z = O.solve_chol(np.zeros((3, 5)), np.array([2.0, 4.0, 6.0, 8.0, 10.0]), 2.0)
    assert np.array_equal(z.x, golden["kat_zero_scores_x"])
    assert np.array_equal(z.x, [1.0, 2.0, 3.0, 4.0, 5.0])


def test_potrf_pivot_kat(golden):
    with pytest.raises(O.OracleFactorizationError) as e:
        O.cholesky_lower(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert e.value.pivot == int(golden["kat_potrf_pivot"][0]) == 1


@pytest.mark.parametrize("name", ["rs_42_8_50", "gp_0_64_4096", "gp_1_100_1000", "gp_2_129_3001", "gp_3_1_7",
                                  "gp_4_16_64", "gp_5_200_20000", "gp_6_40_600", "f32_0_64_4096",
                                  "f32_7_256_32768", "f32_8_300_10000"])
def test_solve_chol_matches_reference(name, golden, manifest):
    S, v, lam = regenerate(manifest["cases"][name])
    sol = O.solve_chol(S, v, lam)
    ref = golden[f"{name}_x"]
    assert np.linalg.norm(sol.x - ref) <= 1e-12 * max(1.0, np.linalg.norm(ref))
    a, r = golden[f"{name}_res"]
    assert abs(sol.rel_residual - r) <= 1e-3 * r + 1e-18
    if f"{name}_W" in golden:
        W = O.gram(S, lam)
        assert np.abs(W - golden[f"{name}_W"]).max() <= 1e-13 * np.abs(W).max()
        L = O.cholesky_lower(W)
        assert np.abs(L - golden[f"{name}_L"]).max() <= 1e-12 * np.abs(L).max()
    u = S @ v
    assert np.abs(u - golden[f"{name}_u"] if f"{name}_u" in golden else 0).max() <= 1e-12 * max(1.0, np.abs(u).max())
    if f"{name}_eigh_x" in golden:
        xe = O.solve_svd_eigh(S, v, lam).x
        xd = O.solve_svd_direct(S, v, lam).x
        assert O.rel_err(xe, golden[f"{name}_eigh_x"]) <= 1e-10
        assert O.rel_err(xd, golden[f"{name}_svd_x"]) <= 1e-10


def test_refinement_branch_is_exercised(manifest):
    # gp_4 / gp_6 have first-pass rel_residual > 1e-10 in the reference -> refinement taken
    for name in ("gp_4_16_64", "gp_6_40_600"):
        S, v, lam = regenerate(manifest["cases"][name])
        assert O.solve_chol(S, v, lam).refined


def test_oracle_agrees_with_dense_lu():
    S, v, lam = O.random_system(42, 8, 50, 1e-3)       # tests/test_solvers.py:93-98
    sol = O.solve_chol(S, v, lam)
    ref = O.dense_solve(S, lam, v)
    assert sol.rel_residual <= 1e-8
    assert np.linalg.norm(sol.x - ref) <= 1e-8 * np.linalg.norm(ref)
