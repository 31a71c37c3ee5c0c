#!/usr/bin/env python
"""Benchmark of the damped-Fisher Cholesky solve (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE configs[1], the paper headline): n=1024 samples, m=1e6 parameters,
fp32 scores, lam=1e-3.  N=1: the reference generator's system (PCG64 seed 0, bench.py:155-160)
rounded to fp32 — the CPU reference solves its exact fp64 upcast, so the line carries
relerr(x) against the reference (`parity`).  One step = one full solve_chol as the drop-in
default runs it on fp32 scores: the f16x2 tensor-core Gram -> potrf -> TRSV pair -> fused
x + y pass -> z-space refinement steps (each one TRSV pair + one fused pass) -> fp64 residual
diagnostics, i.e. the reference's timed unit (solvers.py:151-206 via bench.py:254-267) at the
reference's result quality (rel_residual <= 1e-10, its refinement rule).  `parity` also times
the raw fp32-split modes (no refinement) and the exact fp64 mode on the same system.

N=1: the one-shot C-ABI solve on device-resident inputs (`value`) and the public Python API
with host (pinned) buffers, H2D + D2H inside the timed region (`e2e`; `e2e_streamed_ms` is the
defer=True path that overlaps the upload with the Gram).
N>1 (torchrun, one rank per GPU): the m axis is column-sharded (strong scaling: total m
fixed), one NCCL all-reduce of the packed [W | u] per solve, time = max over ranks.

--impl reference: rank 0 times the CPU oracle port of the reference path (numpy/scipy,
oracle/fisher_oracle.py, all host threads) on the same workload; other ranks exit 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "damped-Fisher solve ms at n=1024,m=1e6; SYRK TC util + GEMV HBM GB/s vs peak"
WORKLOAD = "chol solve n=1024, m=1e6, fp32 scores, lam=1e-3 (BASELINE configs[1], paper headline)"
L2_NOTE = "inputs (S = 4.1 GB fp32) larger than the 126 MB L2; no flush needed"
DATA_NOTE = ("synthetic: the reference generator's system (PCG64 seed 0, S = N(0,1)/sqrt(n) then v, bench.py:155-160) "
             "rounded to fp32; the CPU reference solves its exact fp64 upcast (the identical system)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--m", type=int, default=1_000_000)
    ap.add_argument("--lam", type=float, default=1e-3)
    ap.add_argument("--precision", default="f16x2", choices=["f16x2", "tf32x3", "fp64"])
    ap.add_argument("--refine", default="auto",
                    help="'auto' (the drop-in default: the reference's result rule), or a step count (0 = raw mode)")
    ap.add_argument("--sharded-refine", type=int, default=2,
                    help="z-space refinement steps per solve at N > 1 (fixed: multi-rank control flow is collective)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="run the multi-GPU (column-sharded, NCCL) code path even at one rank (a 1-rank NCCL group)")
    ap.add_argument("--cpu-repeats", type=int, default=2)
    ap.add_argument("--philox", action="store_true", help="device Philox data instead of the reference generator")
    ap.add_argument("--no-modes", dest="modes", action="store_false",
                    help="skip timing the drop-in default and fp64 modes")
    ap.add_argument("--no-pageable", dest="pageable", action="store_false",
                    help="skip timing e2e from pageable numpy memory")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ measured peaks

def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "MEASURED_PEAKS.json (measured)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "B200_PROFILING.md fallback"}


def ncu_traffic(precision):
    """Per-launch DRAM bytes of the SYRK kernel (this precision mode) from the committed ncu
    --set full summary (profiles/ncu_summary.json, written by tools/ncu_summarize.py)."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(f"syrk_tc_kernel:{precision}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------------ clocks during the timed region

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [ln for ln in out.splitlines() if ln.strip()]
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ reference (CPU) arm

def reference_system(n, m, seed=0):
    """The reference generator's system (bench.py:127-171 / SURVEY §8d): PCG64(seed), S = N(0,1)/sqrt(n)
    drawn first in row-major order, then v = N(0,1)^m, both rounded to fp32 for the fp32 workload.
    Returns (S32, v32, S64, v64): the fp32 arrays the GPU solves and their exact fp64 upcasts, the
    identical system the CPU reference solves."""
    import numpy as np
    from oracle import fisher_oracle as O
    S64, v64, _ = O.generate_problem(seed, n, m, 1e-3)
    S32 = S64.astype(np.float32)
    v32 = v64.astype(np.float32)
    np.copyto(S64, S32)            # S64 <- fp64(fp32(S)): same buffer, no second 8 GB array
    v64 = v32.astype(np.float64)
    return S32, v32, S64, v64


def cpu_reference(S64, v64, lam, steps, warmup):
    """Time the oracle port of solve_chol (numpy/scipy, the reference's BLAS/LAPACK calls)."""
    from oracle import fisher_oracle as O
    for _ in range(warmup):
        O.solve_chol(S64, v64, lam)
    times = []
    sol = None
    for _ in range(steps):
        t0 = time.perf_counter()
        sol = O.solve_chol(S64, v64, lam)
        times.append(time.perf_counter() - t0)
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count()
    # one extra, separately timed pass through the oracle's phases (the CPU time next
    # to its gram / potrf / chol_apply (GEMVs + TRSVs) / residual breakdown)
    phases = {}
    t = time.perf_counter()
    W = O.gram(S64, lam)
    phases["gram"] = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    L = O.cholesky_lower(W)
    phases["potrf"] = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    x = O.chol_apply(S64, lam, L, v64)
    phases["chol_apply_gemv_trsv"] = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    O.residual(S64, lam, v64, x)
    phases["residual"] = (time.perf_counter() - t) * 1e3
    cpu_reference.phases_ms = phases
    return times, sol, cores


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    n, m = args.n, args.m
    _, _, S64, v64 = reference_system(n, m)
    warm = max(0, min(args.warmup, 1))
    times, sol, cores = cpu_reference(S64, v64, args.lam, max(1, args.steps), warm)
    ms = statistics.median(times) * 1e3
    line = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus, "steps": len(times),
        "warmup": warm, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": DATA_NOTE,
        "config": {"workload": WORKLOAD, "n": n, "m": m, "lam": args.lam, "l2": L2_NOTE},
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "port",
                         "sample": f"full workload n={n}, m={m} per step, median of {len(times)}",
                         "rel_residual": sol.rel_residual, "phases_ms": getattr(cpu_reference, "phases_ms", None)},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ B200 arm

def make_shard(n, m_local, seed, device, dtype):
    import torch
    g = torch.Generator(device=device).manual_seed(seed)
    per16 = 16 // torch.empty((), dtype=dtype).element_size()
    ld = -(-m_local // per16) * per16
    buf = torch.empty((n, ld), dtype=dtype, device=device)
    S = buf[:, :m_local]
    S.normal_(generator=g).mul_(1.0 / n ** 0.5)
    v = torch.empty(m_local, dtype=dtype, device=device).normal_(generator=g)
    return S, v


def _rel_err(x, ref):
    """||x - ref|| / max(1, ||ref||), the reference's comparison (tests/conftest.py:27-29)."""
    import numpy as np
    return float(np.linalg.norm(np.asarray(x) - ref) / max(1.0, float(np.linalg.norm(ref))))


def run_b200(args, rank, world, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2310_17556_b200 as fsb
    from paper_2310_17556_b200 import _lib
    from paper_2310_17556_b200.distributed import column_shard, sharded_solve_chol_fused

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    sharded = world > 1 or args.sharded
    if sharded:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=device)
    n, m, lam = args.n, args.m, args.lam
    a, b = column_shard(m, world, rank)
    m_local = b - a
    dtype = torch.float64 if args.precision == "fp64" else torch.float32
    S64 = v64 = None
    if world == 1 and not args.philox:
        # N=1: the reference generator's PCG64 system, so x can be compared with the CPU reference
        S32h, v32h, S64, v64 = reference_system(n, m)
        per16 = 16 // torch.empty((), dtype=dtype).element_size()
        ld = -(-m // per16) * per16
        S = torch.empty((n, ld), dtype=dtype, device=device)[:, :m]
        S.copy_(torch.from_numpy(S32h if dtype == torch.float32 else S64))
        v = torch.from_numpy(v32h if dtype == torch.float32 else v64).to(device)
        data = DATA_NOTE
        del S32h
    else:
        S, v = make_shard(n, m_local, 1234 + rank, device, dtype)
        data = ("synthetic: torch Philox N(0,1)/sqrt(n), seed 1234+rank, device-resident (N>1: each rank draws its "
                "own column shard; the CPU-reference comparison runs at N=1)")
    torch.cuda.synchronize()

    ctx = _lib.context_for(local, n, m_local)
    ctx.profile(True)
    system = None
    sm = None
    if not sharded:
        # device-resident public API: ScoreMatrix copies S once into its own aligned device buffer
        # (construction, outside the timed region; the reference copies its array the same way)
        system = fsb.DampedSystem(fsb.ScoreMatrix(S), lam, v)
    else:
        # the shard is validated and aligned once (as the single-GPU DampedSystem is), then every
        # step is one fs_chol_solve per rank with the NCCL all-reduce callback
        sm = fsb.ScoreMatrix(S)

    stage_acc = {k: [] for k in _lib.PROF_STAGES}
    last = {}

    def one_step():
        # the drop-in default on fp32 scores: the f16x2 tensor-core Gram + z-space refinement to the
        # reference's result quality (rel_residual <= 1e-10; solvers.py:41-43, :171-194)
        if not sharded:
            sol = fsb.solve_chol(system, precision=args.precision, refine=args.refine)
        else:
            sol = sharded_solve_chol_fused(sm, v, lam, precision=args.precision, refine=args.sharded_refine)
        for k, val in ctx.stage_ms().items():
            stage_acc[k].append(val)
        last["sol"] = sol
        return sol.rel_residual

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    for k in stage_acc:
        stage_acc[k].clear()

    stream = torch.cuda.current_stream(device)
    launches0 = ctx.launches()
    with ClockSampler(local) as clk:
        if sharded:
            dist.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        rels = [one_step() for _ in range(args.steps)]
        ev1.record(stream)
        torch.cuda.synchronize()
        if sharded:
            dist.barrier()
    launches = ctx.launches() - launches0
    elapsed = ev0.elapsed_time(ev1)
    if sharded:
        t = torch.tensor([elapsed], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    ms_per_step = elapsed / args.steps
    x_head = last["sol"].x_local if sharded else last["sol"].x
    x_head = x_head.cpu().numpy() if isinstance(x_head, torch.Tensor) else np.asarray(x_head)

    # ---- the drop-in defaults and the reference's own arithmetic, timed on the same system (N=1) ----
    modes = {}
    if not sharded and args.modes:
        for name, kw in (("raw f16x2 (no refinement; SURVEY 8d fp32 tolerance relerr <= 1e-6)",
                          dict(precision="f16x2", refine=0)),
                         ("raw tf32x3 (no refinement)", dict(precision="tf32x3", refine=0)),
                         ("fp64 (exact fp64 products, the reference's arithmetic)", dict(precision="fp64"))):
            if dtype == torch.float64 and name.startswith("raw"):
                continue
            sol = fsb.solve_chol(system, **kw)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            reps = 3
            e0.record(stream)
            for _ in range(reps):
                sol = fsb.solve_chol(system, **kw)
            e1.record(stream)
            torch.cuda.synchronize()
            modes[name] = {"ms": e0.elapsed_time(e1) / reps, "precision": sol.precision,
                           "rel_residual": sol.rel_residual, "x": sol.x.cpu().numpy()}
    # ---- the paper's comparison on the same system: chol vs the eigh and svd routes (all GPU) ----
    routes = None
    if not sharded and args.modes:
        routes = {"chol_ms": None}
        for name, fn in (("eigh", fsb.solve_svd_eigh), ("svd", fsb.solve_svd_direct)):
            sol = fn(system)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            reps = 2
            e0.record(stream)
            for _ in range(reps):
                sol = fn(system)
            e1.record(stream)
            torch.cuda.synchronize()
            routes[f"{name}_ms"] = e0.elapsed_time(e1) / reps
            routes[f"{name}_rel_residual"] = sol.rel_residual
            modes[f"route {name}"] = {"ms": routes[f"{name}_ms"], "precision": sol.precision,
                                      "rel_residual": sol.rel_residual, "x": sol.x.cpu().numpy()}

    # ---- end to end through the public API with host buffers ----
    e2e = None
    e2e_extra = {}
    if args.e2e_steps > 0:
        S_host = torch.empty((n, m_local), dtype=dtype, pin_memory=True)
        S_host.copy_(S)
        v_host = torch.empty(m_local, dtype=dtype, pin_memory=True)
        v_host.copy_(v)
        Sh, vh = S_host.numpy(), v_host.numpy()

        def time_e2e(step, steps):
            step()   # warm
            torch.cuda.synchronize()
            if sharded:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            if sharded:
                t = torch.tensor([ms], dtype=torch.float64, device=device)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            return ms

        def e2e_step(host_S, defer=False):
            # the call a user makes with host (numpy) buffers: ScoreMatrix construction uploads and
            # validates S (the reference's frozen copy), the solve returns a numpy x
            if not sharded:
                out = fsb.solve_chol(fsb.DampedSystem(fsb.ScoreMatrix(host_S, defer=defer), lam, vh),
                                     precision=args.precision, refine=args.refine).x
            else:
                out = sharded_solve_chol_fused(fsb.ScoreMatrix(host_S, defer=True), vh, lam,
                                               precision=args.precision, refine=args.sharded_refine).x_local
            assert isinstance(out, np.ndarray)

        e2e_ms = time_e2e(lambda: e2e_step(Sh), args.e2e_steps)
        e2e = {"value": e2e_ms, "unit": "ms",
               "h2d_bytes_per_step": int(Sh.nbytes + vh.nbytes), "d2h_bytes_per_step": int(m_local * 8 + 16),
               "path": ("solve_chol(DampedSystem(ScoreMatrix(pinned numpy S), lam, numpy v)) -> numpy x (the "
                        "drop-in default); construction uploads + validates S on the device"
                        if not sharded else
                        "per rank: sharded_solve_chol_fused(ScoreMatrix(pinned numpy shard, defer=True), numpy v "
                        "shard) -> numpy x shard; max over ranks")}
        if not sharded:
            e2e_extra["e2e_streamed_ms"] = time_e2e(lambda: e2e_step(Sh, defer=True), args.e2e_steps)
            if args.pageable:
                Sp = np.array(Sh)        # ordinary (pageable) numpy memory, what most callers hold
                e2e_extra["e2e_pageable_ms"] = time_e2e(lambda: e2e_step(Sp), max(1, args.e2e_steps - 1))
                del Sp
        del S_host, v_host

    if rank != 0:
        if sharded:
            dist.destroy_process_group()
        return 0

    pk = peaks()
    st = {k: (statistics.median(vals) if vals else None) for k, vals in stage_acc.items()}
    syrk_flops = float(n) * (n + 1) * m_local
    if args.precision == "tf32x3":
        peak_mode = pk["bf16_tflops_sustained"] / 2.0 / 3.0   # tf32 = bf16/2; 3 MMAs per product
        peak_note = "bf16 sustained/2 (tf32) /3 (3xTF32)"
    elif args.precision == "f16x2":
        # the Gram runs inside a multi-ms step: the tensor pipe drives the board into its power cap
        # and the SM clock to ~1.3 GHz (measured in-kernel, FS_SYRK_DBG=256; MEASURED_PEAKS shows
        # the same 1305 MHz under cuBLAS), so the sustained dense figure is the roofline
        peak_mode = pk["bf16_tflops_sustained"] / 3.0      # fp16 = bf16 dense rate; 3 MMAs per product
        peak_note = "bf16 sustained (= fp16 dense, power-capped clocks) /3 (hi*hi + hi*lo + lo*hi)"
    else:
        peak_mode = 36.9                                     # fp64 DMMA, measured (tools/ubench/dmma_peak.cu)
        peak_note = "fp64 DMMA 36.9 TF/s measured (tools/ubench/dmma_peak.cu)"
    roofline = None
    if st.get("gram"):
        achieved = syrk_flops / (st["gram"] * 1e-3) / 1e12
        burst = peak_mode * pk["bf16_tflops"] / pk["bf16_tflops_sustained"] if args.precision != "fp64" else None
        roofline = {"bound": "tensor", "kernel": "syrk_tc_kernel (+split-K reduce)", "achieved": achieved,
                    "peak": peak_mode, "unit": "TFLOP/s", "frac": achieved / peak_mode,
                    "frac_vs_burst_peak": (achieved / burst) if burst else None,
                    "traffic": ncu_traffic(args.precision), "flops_per_launch": syrk_flops,
                    "peak_source": f"{pk['source']}: {peak_note}"}
    es = dtype.itemsize
    gemv = {}
    if st.get("gemv_sv"):
        # K3 by SURVEY §8(d): n m s + m s + n 8 (read S and v once, write u); the retile pass also
        # writes the tiled copy (F16X2: two fp16 planes, 4 bytes per score) -> both figures
        tiles = (-(-n // 256) * 256) * (-(-m_local // 64) * 64) * 4 if args.precision != "fp64" else 0
        bytes_k3 = n * m_local * es + m_local * es + n * 8
        gemv["gemv_sv_GBps"] = bytes_k3 / (st["gemv_sv"] * 1e-3) / 1e9
        gemv["gemv_sv_with_tile_write_GBps"] = (bytes_k3 + tiles) / (st["gemv_sv"] * 1e-3) / 1e9
    if st.get("gemv_stz"):
        # fused x = (v - S^T z)/lam and y = S x (cluster kernel): S from HBM exactly once
        bytes_stz = n * m_local * es + m_local * es + m_local * 8 + n * 8
        gemv["gemv_stz_GBps"] = bytes_stz / (st["gemv_stz"] * 1e-3) / 1e9
    if st.get("residual"):
        bytes_res = n * m_local * es + m_local * (es + 8) + n * 8
        gemv["residual_GBps"] = bytes_res / (st["residual"] * 1e-3) / 1e9
    if gemv:
        gemv = {"bound": "hbm", "peak": pk["hbm_gbs"], "unit": "GB/s",
                **gemv, **{k.replace("GBps", "frac"): val / pk["hbm_gbs"] for k, val in list(gemv.items())}}

    cpu = None
    parity = None
    if world == 1 and S64 is not None and not args.no_cpu_baseline:
        try:
            times, sol_ref, cores = cpu_reference(S64, v64, lam, args.cpu_repeats, 0)
            cpu = {"value": statistics.median(times) * 1e3, "unit": "ms", "cores": cores, "kind": "port",
                   "sample": f"full workload n={n}, m={m_local} fp64 oracle solve_chol on the identical system, "
                             f"median of {len(times)}",
                   "rel_residual": sol_ref.rel_residual, "phases_ms": getattr(cpu_reference, "phases_ms", None)}
            parity = {"tolerance_relerr_fp32_modes": 1e-6, "tolerance_relerr_fp64": 1e-10,
                      "reference_rel_residual": sol_ref.rel_residual,
                      "headline": {"precision": args.precision, "refine": str(args.refine),
                                   "rel_residual": rels[-1], "reference_gate_1e-6": rels[-1] <= 1e-6,
                                   "relerr_vs_reference": _rel_err(x_head, sol_ref.x)}}
            for name, d in modes.items():
                parity[name] = {"ms": d["ms"], "precision": d["precision"], "rel_residual": d["rel_residual"],
                                "relerr_vs_reference": _rel_err(d["x"], sol_ref.x)}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "ms", "cores": None, "kind": "port", "sample": f"failed: {e}"}

    line = {
        "metric": METRIC, "value": ms_per_step, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if dtype == torch.float32 else "f64",
        "data": data,
        "config": {"workload": WORKLOAD, "n": n, "m": m, "m_per_rank": m_local, "lam": lam,
                   "precision": args.precision,
                   "refine": (f"{args.refine} (z-space refinement: f16x2 factor, exact fp64 residuals)"
                              if args.precision != "fp64" else f"{args.refine} (the reference's rule)"),
                   "diagnostics": True, "l2": L2_NOTE,
                   "parallelism": f"column-shard m over {world} GPU(s), NCCL all-reduce of [W|u]"},
        "roofline": roofline,
        "roofline_gemv": gemv or None,
        "stage_ms": st,
        "routes": routes if routes is None else {**routes, "chol_ms": ms_per_step,
                                                 "note": "solve_svd_eigh / solve_svd_direct with their defaults on "
                                                         "the same device-resident system (paper: chol vs eigh/svda)"},
        "rel_residual": rels[-1],
        "parity": parity,
        "cpu_baseline": cpu,
        "e2e": e2e,
        **e2e_extra,
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.refine != "auto":
        args.refine = int(args.refine)
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_b200(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
