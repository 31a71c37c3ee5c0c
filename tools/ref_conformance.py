"""Run the reference package's OWN test suite against the B200 drop-in (SURVEY §8c protocol).

    python tools/ref_conformance.py [--out profiles/r02_ref_conformance.json] [-k EXPR]

The reference (``fisher_solve``) and its tests are test infrastructure here, installed outside
the product and outside git history: ``baseline/_ref`` holds the ``pip install --target`` of
/root/reference/pkg (the one offline install the task allows) and ``baseline/_ref/tests`` a copy
of its test files (``baseline/_ref`` is git-ignored, not gpurun-ignored, so it travels to the GPU
box).  Nothing under ``paper_2310_17556_b200/`` imports any of it.

A shim module named ``fisher_solve`` is installed in ``sys.modules`` before the tests are
collected: every name the B200 package provides (ScoreMatrix, DampedSystem, gram, residual,
solve_chol*, the eigh / svd routes, ThinSvd, CholWorkspace, _cholesky_lower, resolve_solver, FMAT
I/O, the CLI ...) is the B200 one — exactly the swap a user makes — and only the reference's
CPU-only baselines that are out of this package's scope (solve_naive, solve_cg, solve_rvb, the
SR adapters, the timing harness) stay the reference's, serving as the tests' oracles.  The B200
entry points accept the reference's objects (as_system / as_scores), so fixtures built by the
reference's generate_problem flow straight into the GPU path.  Tolerances are the reference's,
unchanged.  Writes a per-test JSON summary.
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import os
import sys
import time
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PKG = os.path.join(ROOT, "baseline", "_ref", "fisher_solve")
REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "tests")

# Reference tests that cannot pass against the drop-in, each for a stated out-of-scope reason
# (run with --all: everything else must pass).  The CPU-only baselines (naive / cg / rvb) and the
# timing harness stay the reference's own code behind the shim; where such a test compares the
# reference's enum members with the shim's (the B200 package defines its own Method / Variant),
# identity fails although the values agree.
OUT_OF_SCOPE = {
    "test_acceptance.py::test_criterion_6_scaling_exponents":
        "fits CPU-timing exponents (vary-m >= 0.7); the GPU solve is launch-latency bound at its small m",
    "test_bench.py::TestTimeMethod::test_method_accepts_strings": "enum identity: reference harness vs shim Method",
    "test_bench.py::TestTimeMethod::test_rvb_timed_with_structured_problem": "rvb baseline (CPU-only, out of scope)",
    "test_bench.py::TestResolveSolver::test_every_method_resolves_on_suitable_input":
        "resolve_solver raises for the CPU-only baselines naive / cg / rvb (no CPU fallback in the product)",
    "test_cli.py::TestSolve::test_rvb_reads_coefficients_as_rhs": "rvb baseline (CPU-only, out of scope)",
    "test_cli.py::TestBench::test_structured_bench_can_time_rvb": "rvb baseline (CPU-only, out of scope)",
    "test_cli.py::TestCheck::test_passes_on_well_posed_problem":
        "`check` compares 7 methods incl. naive / cg / rvb; the B200 CLI checks chol / eigh / svd and variants (6 lines)",
    "test_solvers.py::TestSolveNaive::test_hermitian_variant": "enum identity: reference naive vs shim Variant",
    "test_solvers.py::TestSolveRvb::test_hand_example": "enum identity: reference rvb vs shim Method",
}

# the reference suites of the drop-in boundary (VERDICT r1 "next round" #3)
SELECTION = [
    "test_core.py",
    "test_solvers.py::TestSolveChol",
    "test_solvers.py::TestSolveCholHermitian",
    "test_solvers.py::TestSolveRealpart",
    "test_solvers.py::TestThinSvdEigh",
    "test_solvers.py::TestThinSvdDirect",
    "test_solvers.py::TestSolveSvdFromFactors",
    "test_solvers.py::TestSolveSvdWrappers",
    "test_solvers.py::TestCholeskyMachinery",
    "test_solvers.py::TestCrossMethodProperties",
    "test_acceptance.py::test_criterion_1_oracle_equivalence",
    "test_acceptance.py::test_criterion_2_factored_route_satisfies_original_system",
    "test_acceptance.py::test_criterion_4_complex_variants",
    "test_acceptance.py::test_criterion_8_memory_contract",
    "test_acceptance.py::test_criterion_9_degenerate_cases",
    "test_acceptance.py::test_criterion_10_fmat_round_trip",
    "test_acceptance.py::test_criterion_7_method_ordering",
    "test_fmat.py",
]


def load_reference():
    spec = importlib.util.spec_from_file_location("fisher_solve_ref", os.path.join(REF_PKG, "__init__.py"),
                                                  submodule_search_locations=[REF_PKG])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["fisher_solve_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def install_shim():
    sys.path.insert(0, ROOT)
    import paper_2310_17556_b200 as fsb
    from paper_2310_17556_b200 import cli as b_cli, core as b_core, fmat as b_fmat, solvers as b_solvers
    ref = load_reference()
    for sub in ("core", "solvers", "fmat", "cli", "bench", "sr"):
        importlib.import_module(f"fisher_solve_ref.{sub}")
    provided = {}

    def overlay(name, ref_mod, *ours):
        m = types.ModuleType(name)
        for k in dir(ref_mod):
            if k.startswith("__"):
                continue
            for o in ours:
                if hasattr(o, k):
                    setattr(m, k, getattr(o, k))
                    provided.setdefault(name, []).append(k)
                    break
            else:
                setattr(m, k, getattr(ref_mod, k))
        return m

    shim = overlay("fisher_solve", ref, fsb, b_solvers, b_core, b_fmat)
    shim.__path__ = []
    subs = {
        "core": overlay("fisher_solve.core", ref.core, b_core, fsb),
        "solvers": overlay("fisher_solve.solvers", ref.solvers, b_solvers, fsb),
        "fmat": overlay("fisher_solve.fmat", ref.fmat, b_fmat),
        "cli": overlay("fisher_solve.cli", ref.cli, b_cli),
        "bench": ref.bench,     # the timing harness (out of scope) calls the B200 solvers through the shim
        "sr": ref.sr,
    }
    # the reference's harness resolves solvers from its own module namespace: point it at ours
    for k in ("solve_chol", "solve_chol_hermitian", "solve_realpart", "solve_svd_eigh", "solve_svd_direct"):
        setattr(ref.bench, k, getattr(b_solvers, k))
    sys.modules["fisher_solve"] = shim
    for k, v in subs.items():
        sys.modules[f"fisher_solve.{k}"] = v
        setattr(shim, k, v)
    return provided


class Collector:
    def __init__(self):
        self.results = {}

    def pytest_runtest_logreport(self, report):
        if report.when == "call" or (report.when == "setup" and report.outcome != "passed"):
            entry = {"outcome": report.outcome, "seconds": round(report.duration, 3)}
            if report.outcome == "failed":
                lines = str(report.longrepr).splitlines()
                err = [ln for ln in lines if ln.startswith("E ")]
                entry["error"] = (" | ".join(err[:6]) + " @ " + lines[-1])[:1200]
            self.results[report.nodeid] = entry


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_ref_conformance.json"))
    ap.add_argument("-k", default=None)
    ap.add_argument("--all", action="store_true", help="run every reference test file")
    args = ap.parse_args()
    if not os.path.isdir(REF_PKG) or not os.path.isdir(REF_TESTS):
        print(f"reference not staged under {REF_PKG} / {REF_TESTS}", file=sys.stderr)
        return 2
    import pytest
    provided = install_shim()
    sys.path.insert(0, REF_TESTS)
    targets = [os.path.join(REF_TESTS, t) for t in SELECTION] if not args.all else [REF_TESTS]
    col = Collector()
    t0 = time.time()
    argv = ["-q", "-p", "no:cacheprovider", "--rootdir", REF_TESTS, "-o", "python_files=test_*.py", *targets]
    if args.k:
        argv += ["-k", args.k]
    rc = pytest.main(argv, plugins=[col])
    counts = {}
    for r in col.results.values():
        counts[r["outcome"]] = counts.get(r["outcome"], 0) + 1
    import torch
    summary = {
        "what": "the reference's own tests (baseline/_ref/tests, unchanged tolerances) run against the B200 "
                "drop-in through a fisher_solve shim (tools/ref_conformance.py)",
        "selection": SELECTION if not args.all else "all",
        "b200_names": provided,
        "device": torch.cuda.get_device_name(0) if torch.cuda.is_available() else None,
        "pytest_exit": int(rc), "counts": counts, "seconds": round(time.time() - t0, 1),
        "failures_outside_the_out_of_scope_list": sorted(k for k, r in col.results.items()
                                                         if r["outcome"] != "passed" and k not in OUT_OF_SCOPE),
        "out_of_scope": OUT_OF_SCOPE if args.all else None,
        "tests": col.results,
    }
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({"counts": counts, "exit": int(rc)}))
    return 0 if rc == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
