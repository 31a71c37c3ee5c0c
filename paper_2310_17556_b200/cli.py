"""GPU command line tool, the counterpart of fisher_solve/cli.py:1-294.

    python -m paper_2310_17556_b200.cli gen     --n N --m M [--kind real|complex|structured] --out PREFIX
    python -m paper_2310_17556_b200.cli solve   S.fmat v.fmat --method chol|eigh|svd [--variant ...] [--out x.fmat]
    python -m paper_2310_17556_b200.cli bench   --n N --m M --method chol [--precision auto|fp64|f16x2|tf32x3]
    python -m paper_2310_17556_b200.cli scaling --method chol --fix n=1024 --vary m=1e5:1e6:4
    python -m paper_2310_17556_b200.cli check   --n N --m M

Same subcommands, flags, CSV schema (bench.py:38) and exit codes as the reference for the methods
this package runs on the GPU (chol with the plain/hermitian/realpart variants, eigh, svd); the
CPU-only baselines (naive, rvb, cg) are not provided and are rejected by argparse.  FMAT inputs
are read straight into page-locked memory, so ``solve`` streams S to the device through the
pipelined host entry.  ``check`` cross-validates the GPU routes against a dense GPU solve of the
m x m system (small m) and against each other.
"""

from __future__ import annotations

import argparse
import os
import enum
import math
import statistics
import sys
import time

import numpy as np

from . import fmat

CSV_HEADER = "method,n,m,lambda,seed,repeats,median_s,min_s,rel_residual,status"
REL_RESIDUAL_GATE = 1e-6       # bench.py:40
_MAX_PROBLEM_BYTES = 1 << 34   # bench.py:42
_METHODS = ("chol", "eigh", "svd")
_VARIANTS = ("plain", "hermitian", "realpart")
_PRECISIONS = ("auto", "fp64", "f16x2", "tf32x3")


class Kind(enum.Enum):
    REAL_GAUSSIAN = "real"
    COMPLEX_GAUSSIAN = "complex"
    STRUCTURED = "structured"


def generate_problem(seed: int, n: int, m: int, lam: float, kind: str = "real"):
    """Seeded problem with the reference generator's stream layout (bench.py:127-171): PCG64(seed);
    scores N(0,1)/sqrt(n) in row-major order (complex: the whole real block, then the imaginary
    block), then v (structured: f ~ N(0,1)^n and v = S^T f).  Returns (S, v, lam, f or None)."""
    n, m, seed = int(n), int(m), int(seed)
    if n < 1 or m < 1:
        raise ValueError(f"problem needs n >= 1 and m >= 1, got {n}x{m}")
    kind = Kind(kind)
    if n * m * (16 if kind is Kind.COMPLEX_GAUSSIAN else 8) > _MAX_PROBLEM_BYTES:
        raise ValueError(f"refusing to generate a {n}x{m} problem beyond {_MAX_PROBLEM_BYTES} bytes of scores")
    g = np.random.Generator(np.random.PCG64(seed))
    root_n = math.sqrt(float(n))            # divide (not multiply by 1/sqrt(n)): bit-identical draws
    f = None
    if kind is Kind.COMPLEX_GAUSSIAN:
        re = g.standard_normal((n, m))
        im = g.standard_normal((n, m))
        S = (re + 1j * im) / root_n
        v = g.standard_normal(m) + 1j * g.standard_normal(m)
    else:
        S = g.standard_normal((n, m)) / root_n
        if kind is Kind.REAL_GAUSSIAN:
            v = g.standard_normal(m)
        else:
            f = g.standard_normal(n)
            v = f @ S
    return S, v, float(lam), f


def _solver(method: str, variant: str):
    import paper_2310_17556_b200 as fsb
    if method == "chol":
        return {"plain": fsb.solve_chol, "hermitian": fsb.solve_chol_hermitian,
                "realpart": fsb.solve_realpart}[variant]
    if variant != "plain":
        raise ValueError(f"method {method} supports the plain variant only")
    return fsb.solve_svd_eigh if method == "eigh" else fsb.solve_svd_direct


def _run(system, method, variant, precision, refine=None):
    f = _solver(method, variant)
    kw = {"precision": precision}
    if refine is not None and method == "chol":
        kw["refine"] = refine
    return f(system, **kw)


def _parse_refine(text):
    if text in ("auto", None):
        return "auto"
    if text in ("true", "false"):
        return text == "true"
    return int(text)


def _cmd_gen(args) -> int:
    S, v, _, f = generate_problem(args.seed, args.n, args.m, args.lam, args.kind)
    paths = [args.out + ".S.fmat", args.out + ".v.fmat"]
    fmat.write_matrix(paths[0], S)
    fmat.write_vector(paths[1], v)
    if f is not None:
        paths.append(args.out + ".f.fmat")
        fmat.write_vector(paths[2], f)
    print(f"wrote {', '.join(paths)} ({args.n}x{args.m} {args.kind}, seed {args.seed})")
    return 0


def _cmd_solve(args) -> int:
    import paper_2310_17556_b200 as fsb
    S = fmat.read_matrix(args.scores)            # page-locked
    rhs = fmat.read_vector(args.rhs)
    if args.precision != "fp64" and not np.iscomplexobj(S) and args.fp32:
        S = S.astype(np.float32)
        rhs = rhs.astype(np.float32)
    system = fsb.DampedSystem(fsb.ScoreMatrix(S, defer=True), args.lam, rhs)
    sol = _run(system, args.method, args.variant, args.precision, _parse_refine(args.refine))
    if args.out is not None:
        fmat.write_vector(args.out, sol.x)
    print(f"method={args.method} n={S.shape[0]} m={S.shape[1]} lambda={args.lam!r} "
          f"rel_residual={sol.rel_residual:.3e} wall_s={sol.wall_seconds:.6f} precision={sol.precision}")
    return 0


def _time(system, method, variant, precision, warmup, repeats):
    import torch
    for _ in range(max(0, warmup)):
        _run(system, method, variant, precision)
    times, sol = [], None
    for _ in range(repeats):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sol = _run(system, method, variant, precision)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    return times, sol


def _record(method, n, m, lam, seed, repeats, times, sol) -> str:
    status = "ok" if sol is not None and sol.rel_residual <= REL_RESIDUAL_GATE else "residual"
    med = statistics.median(times)
    return ",".join([method, str(n), str(m), repr(lam), str(seed), str(repeats), f"{med:.6e}", f"{min(times):.6e}",
                     f"{sol.rel_residual:.6e}", status])


def _system_for(args, n, m):
    import paper_2310_17556_b200 as fsb
    import torch
    S, v, lam, _ = generate_problem(args.seed, n, m, args.lam, getattr(args, "kind", "real"))
    if args.precision in ("f16x2", "tf32x3") or (args.precision == "auto" and args.fp32):
        S = S.astype(np.complex64 if np.iscomplexobj(S) else np.float32)
        v = v.astype(np.complex64 if np.iscomplexobj(v) else np.float32)
    if args.device_resident:
        dev = torch.device("cuda", torch.cuda.current_device())
        return fsb.DampedSystem(fsb.ScoreMatrix(torch.from_numpy(S).to(dev)), lam, torch.from_numpy(v).to(dev))
    return fsb.DampedSystem(fsb.ScoreMatrix(S, defer=True), lam, v)


def _cmd_bench(args) -> int:
    system = _system_for(args, args.n, args.m)
    if args.variant == "realpart":
        import paper_2310_17556_b200 as fsb
        system = fsb.DampedSystem(system.S, system.lam, system.v_tensor.real.contiguous())
    times, sol = _time(system, args.method, args.variant, args.precision, args.warmup, args.repeats)
    print(CSV_HEADER)
    row = _record(args.method, args.n, args.m, args.lam, args.seed, args.repeats, times, sol)
    print(row)
    return 0 if row.endswith(",ok") else 1


def _cmd_scaling(args) -> int:
    fix_name, fix_size = args.fix
    vary_name, sizes = args.vary
    if fix_name == vary_name:
        raise ValueError(f"--fix and --vary target the same dimension {fix_name!r}")
    print(CSV_HEADER)
    xs, ys = [], []
    for size in sizes:
        n = size if vary_name == "n" else fix_size
        m = size if vary_name == "m" else fix_size
        times, sol = _time(_system_for(args, n, m), args.method, "plain", args.precision, args.warmup, args.repeats)
        print(_record(args.method, n, m, args.lam, args.seed, args.repeats, times, sol))
        xs.append(math.log(size))
        ys.append(math.log(statistics.median(times)))
    k = len(xs)
    mx, my = sum(xs) / k, sum(ys) / k
    sxx = sum((x - mx) ** 2 for x in xs)
    slope = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sxx
    ss_res = sum((y - (my + slope * (x - mx))) ** 2 for x, y in zip(xs, ys))
    ss_tot = sum((y - my) ** 2 for y in ys) or 1.0
    print(f"# scaling {vary_name} in [{sizes[0]}, {sizes[-1]}] at {fix_name}={fix_size}: "
          f"exponent={slope:.3f} r_squared={1 - ss_res / ss_tot:.4f}")
    return 0


def _dense_solve(S, lam, v, variant):
    """Dense m x m reference solve on the GPU (check only; small m)."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    A = torch.from_numpy(np.ascontiguousarray(S)).to(dev)
    vt = torch.from_numpy(np.ascontiguousarray(v)).to(dev)
    if variant == "plain":
        M = A.T @ A
    elif variant == "hermitian":
        M = A.conj().T @ A
    else:
        M = (A.real.T @ A.real + A.imag.T @ A.imag)
    M = M + lam * torch.eye(M.shape[0], dtype=M.dtype, device=dev)
    return torch.linalg.solve(M, vt.to(M.dtype)).cpu().numpy()


def _cmd_check(args) -> int:
    import paper_2310_17556_b200 as fsb
    tol, failures = args.tol, 0

    def rel(x, ref):
        return float(np.linalg.norm(x - ref) / max(1.0, np.linalg.norm(ref)))

    def report(label, err):
        nonlocal failures
        ok = err <= tol
        failures += 0 if ok else 1
        print(f"{'ok  ' if ok else 'FAIL'} {label}: relative error {err:.3e}")

    if args.m > 8192:
        raise ValueError("check builds the dense m x m system on the GPU; use m <= 8192")
    S, v, lam, _ = generate_problem(args.seed, args.n, args.m, args.lam)
    real = fsb.DampedSystem(fsb.ScoreMatrix(S), lam, v)
    dense = _dense_solve(S, lam, v, "plain")
    report("chol vs dense", rel(fsb.solve_chol(real).x, dense))
    report("eigh vs dense", rel(fsb.solve_svd_eigh(real).x, dense))
    report("svd vs dense", rel(fsb.solve_svd_direct(real).x, dense))
    S32 = fsb.DampedSystem(fsb.ScoreMatrix(S.astype(np.float32)), lam, v.astype(np.float32))
    dense32 = _dense_solve(S.astype(np.float32).astype(np.float64), lam, v.astype(np.float32).astype(np.float64),
                           "plain")
    err32 = rel(fsb.solve_chol(S32, refine=8).x, dense32)
    report("chol f16x2 + refinement vs dense (fp32-rounded system)", err32)
    Sc, vc, _, _ = generate_problem(args.seed, args.n, args.m, args.lam, "complex")
    herm = fsb.DampedSystem(fsb.ScoreMatrix(Sc), lam, vc)
    report("hermitian chol vs dense", rel(fsb.solve_chol_hermitian(herm).x, _dense_solve(Sc, lam, vc, "hermitian")))
    rp = fsb.DampedSystem(fsb.ScoreMatrix(Sc), lam, vc.real.copy())
    report("realpart chol vs dense", rel(fsb.solve_realpart(rp).x, _dense_solve(Sc, lam, vc.real.copy(), "realpart")))
    print("all checks passed" if failures == 0 else f"{failures} check(s) failed")
    return 0 if failures == 0 else 1


def _parse_fix(text: str):
    name, _, value = text.partition("=")
    if name not in ("n", "m") or not value:
        raise ValueError(f"--fix expects n=<int> or m=<int>, got {text!r}")
    size = int(float(value))
    if size < 1:
        raise ValueError(f"--fix size must be >= 1, got {size}")
    return name, size


def _parse_vary(text: str):
    name, _, sweep = text.partition("=")
    parts = sweep.split(":")
    if name not in ("n", "m") or len(parts) != 3:
        raise ValueError(f"--vary expects n|m=START:STOP:COUNT, got {text!r}")
    start, stop, count = (int(float(p)) for p in parts)
    if start < 1 or stop < start or count < 3:
        raise ValueError("--vary needs START >= 1, STOP >= START, COUNT >= 3")
    return name, sorted({int(round(s)) for s in np.geomspace(start, stop, count)})


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="fisher-solve-b200",
                                description="Solve and benchmark (S^T S + lambda I) x = v on a B200.")
    sub = p.add_subparsers(dest="command", required=True)

    def problem(sp, kind=True):
        sp.add_argument("--n", type=int, required=True)
        sp.add_argument("--m", type=int, required=True)
        sp.add_argument("--lambda", dest="lam", type=float, default=1e-3)
        sp.add_argument("--seed", type=int, default=0)
        if kind:
            sp.add_argument("--kind", choices=[k.value for k in Kind], default="real")

    def gpu(sp):
        sp.add_argument("--precision", choices=_PRECISIONS, default="auto")
        sp.add_argument("--fp32", action="store_true", help="round the scores to float32 (tensor-core modes)")
        sp.add_argument("--device-resident", action="store_true", help="time with S already in HBM")

    g = sub.add_parser("gen", help="write a seeded problem to FMAT files")
    problem(g)
    g.add_argument("--out", required=True, metavar="PREFIX")
    g.set_defaults(func=_cmd_gen)

    s = sub.add_parser("solve", help="read FMAT inputs, solve on the GPU, write FMAT x")
    s.add_argument("scores")
    s.add_argument("rhs")
    s.add_argument("--lambda", dest="lam", type=float, default=1e-3)
    s.add_argument("--method", choices=_METHODS, required=True)
    s.add_argument("--variant", choices=_VARIANTS, default="plain")
    s.add_argument("--refine", default="auto", help="auto | true | false | <steps> (chol only)")
    s.add_argument("--precision", choices=_PRECISIONS, default="auto")
    s.add_argument("--fp32", action="store_true", help="round real scores to float32 (tensor-core modes)")
    s.add_argument("--out", default=None, metavar="PATH")
    s.set_defaults(func=_cmd_solve)

    b = sub.add_parser("bench", help="time one method on one generated problem")
    problem(b)
    b.add_argument("--method", choices=_METHODS, required=True)
    b.add_argument("--variant", choices=_VARIANTS, default="plain")
    b.add_argument("--repeats", type=int, default=5)
    b.add_argument("--warmup", type=int, default=2)
    gpu(b)
    b.set_defaults(func=_cmd_bench)

    sc = sub.add_parser("scaling", help="sweep one dimension and fit the scaling exponent")
    sc.add_argument("--method", choices=_METHODS, required=True)
    sc.add_argument("--fix", type=_parse_fix, required=True)
    sc.add_argument("--vary", type=_parse_vary, required=True)
    sc.add_argument("--lambda", dest="lam", type=float, default=1e-3)
    sc.add_argument("--seed", type=int, default=0)
    sc.add_argument("--repeats", type=int, default=5)
    sc.add_argument("--warmup", type=int, default=2)
    gpu(sc)
    sc.set_defaults(func=_cmd_scaling)

    c = sub.add_parser("check", help="cross-validate the GPU routes against a dense GPU solve")
    problem(c, kind=False)
    c.add_argument("--tol", type=float, default=1e-7)
    c.set_defaults(func=_cmd_check)
    return p


def _thread_limit():
    """FISHER_SOLVE_THREADS (cli.py:259-266): host-thread cap, 0 or unset = automatic; a negative
    value is an error.  Here it caps the host-side threads (torch's CPU pool), the GPU is unaffected."""
    raw = os.environ.get("FISHER_SOLVE_THREADS", "").strip()
    if not raw:
        return None
    limit = int(raw)
    if limit < 0:
        raise ValueError(f"FISHER_SOLVE_THREADS must be >= 0, got {limit}")
    return limit or None


def run_cli(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return exc.code if isinstance(exc.code, int) else 2
    from .core import FactorizationError
    try:
        limit = _thread_limit()
        if limit is not None:
            import torch
            torch.set_num_threads(limit)
        return args.func(args)
    except (ValueError, OSError, FactorizationError) as exc:
        print(f"fisher-solve-b200: error: {exc}", file=sys.stderr)
        return 1


def main() -> None:
    sys.exit(run_cli())


if __name__ == "__main__":
    main()
