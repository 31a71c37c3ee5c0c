"""Shared fixtures.  `-m gpu` tests need a CUDA device and the built libfisher_b200.so;
everything else runs on CPU (oracle vs golden fixtures, ABI surface, gloo sharding)."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(GOLDEN))


@pytest.fixture(scope="session")
def manifest():
    import json
    with open(os.path.join(ROOT, "tests", "golden", "MANIFEST.json")) as f:
        return json.load(f)


def regenerate(case):
    """Rebuild a golden case's inputs with the oracle's generator restatement."""
    from oracle import fisher_oracle as O
    if case["gen"] == "random_system":
        S, v, lam = O.random_system(case["seed"], case["n"], case["m"], case["lam"])
    elif case["gen"] == "generate_problem+complex":
        return O.generate_problem_complex(case["seed"], case["n"], case["m"], case["lam"])
    else:
        S, v, lam = O.generate_problem(case["seed"], case["n"], case["m"], case["lam"])
    if case["gen"].endswith("+f32"):
        S = S.astype(np.float32).astype(np.float64)
        v = v.astype(np.float32).astype(np.float64)
    return S, v, lam
