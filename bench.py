#!/usr/bin/env python
"""Benchmark of the damped-Fisher Cholesky solve (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

Workload (BASELINE configs[1], the paper headline): n=1024 samples, m=1e6 parameters,
fp32 scores, lam=1e-3, synthetic N(0,1)/sqrt(n) (torch Philox, seed 0 + rank).  One step =
one full solve_chol (Gram -> potrf -> TRSV pair -> fused x epilogue -> fp64 residual
diagnostics), i.e. the reference's timed unit (solvers.py:151-206 via bench.py:254-267).

N=1: the one-shot C-ABI solve on device-resident inputs (`value`) and the public Python API
with host (pinned) buffers, H2D + D2H inside the timed region (`e2e`).
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
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="run the multi-GPU (column-sharded, NCCL) code path even at one rank (a 1-rank NCCL group)")
    ap.add_argument("--cpu-repeats", type=int, default=2)
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

def cpu_reference(n, m, lam, steps, warmup, seed=0):
    """Time the oracle port of solve_chol (numpy/scipy, the reference's BLAS/LAPACK calls)."""
    import numpy as np
    from oracle import fisher_oracle as O
    rng = np.random.Generator(np.random.PCG64(seed))
    S = (rng.standard_normal((n, m), dtype=np.float32) / np.float32(np.sqrt(n))).astype(np.float64)
    v = rng.standard_normal(m, dtype=np.float32).astype(np.float64)
    for _ in range(warmup):
        O.solve_chol(S, v, lam)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        sol = O.solve_chol(S, v, lam)
        times.append(time.perf_counter() - t0)
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count()
    # one extra, separately timed pass through the oracle's phases (the CPU time next
    # to its gram / potrf / chol_apply (GEMVs + TRSVs) / residual breakdown)
    phases = {}
    t = time.perf_counter()
    W = O.gram(S, lam)
    phases["gram"] = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    L = O.cholesky_lower(W)
    phases["potrf"] = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    x = O.chol_apply(S, lam, L, v)
    phases["chol_apply_gemv_trsv"] = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    O.residual(S, lam, v, x)
    phases["residual"] = (time.perf_counter() - t) * 1e3
    cpu_reference.phases_ms = phases
    return times, sol.rel_residual, cores


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    n, m = args.n, args.m
    times, rel, cores = cpu_reference(n, m, args.lam, max(1, args.steps), max(0, min(args.warmup, 1)))
    ms = statistics.median(times) * 1e3
    line = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": args.gpus, "steps": len(times),
        "warmup": max(0, min(args.warmup, 1)), "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": "synthetic: PCG64 N(0,1)/sqrt(n) rounded to fp32, upcast to fp64 (the identical system)",
        "config": {"workload": WORKLOAD, "n": n, "m": m, "lam": args.lam, "l2": L2_NOTE},
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": cores, "kind": "port",
                         "sample": f"full workload n={n}, m={m} per step, median of {len(times)}",
                         "rel_residual": rel, "phases_ms": getattr(cpu_reference, "phases_ms", None)},
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
    S, v = make_shard(n, m_local, 1234 + rank, device, dtype)
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

    def one_step():
        if not sharded:
            sol = fsb.solve_chol(system, precision=args.precision)
            for k, val in ctx.stage_ms().items():
                stage_acc[k].append(val)
            return sol.rel_residual
        sol = sharded_solve_chol_fused(sm, v, lam, precision=args.precision)
        for k, val in ctx.stage_ms().items():
            stage_acc[k].append(val)
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

    # ---- end to end through the public API with host buffers (N=1, rank 0) ----
    e2e = None
    if args.e2e_steps > 0:
        S_host = torch.empty((n, m_local), dtype=dtype, pin_memory=True)
        S_host.copy_(S)
        v_host = torch.empty(m_local, dtype=dtype, pin_memory=True)
        v_host.copy_(v)
        Sh, vh = S_host.numpy(), v_host.numpy()

        def e2e_step():
            # the call a user makes with host (numpy) buffers: the single-GPU public API, or per rank
            # the sharded one (same pipelined host entry + the NCCL all-reduce callback)
            if not sharded:
                out = fsb.solve_chol(fsb.DampedSystem(fsb.ScoreMatrix(Sh), lam, vh), precision=args.precision).x
            else:
                out = sharded_solve_chol_fused(fsb.ScoreMatrix(Sh), vh, lam, precision=args.precision).x_local
            assert isinstance(out, np.ndarray)

        e2e_step()   # warm
        torch.cuda.synchronize()
        if sharded:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1) / args.e2e_steps
        if sharded:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": e2e_ms, "unit": "ms",
               "h2d_bytes_per_step": int(Sh.nbytes + vh.nbytes), "d2h_bytes_per_step": int(m_local * 8 + 16),
               "path": ("solve_chol(DampedSystem(ScoreMatrix(pinned numpy S), lam, numpy v)) -> numpy x"
                        if not sharded else
                        "per rank: sharded_solve_chol_fused(ScoreMatrix(pinned numpy shard), numpy v shard) -> numpy x"
                        " shard; max over ranks")}
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
        peak_mode = 40.0                                     # fp64 (nominal B200 FP64)
        peak_note = "nominal B200 fp64 40 TF/s"
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
        # tf32x3: the retile pass reads S once and writes the tiled copy S_t (tiles.cuh) + u = S v
        tiles = (-(-n // 256) * 256) * (-(-m_local // 64) * 64) * 4 if args.precision != "fp64" else 0
        bytes_sv = n * m_local * es + tiles + m_local * es + n * 8
        gemv["gemv_sv_GBps"] = bytes_sv / (st["gemv_sv"] * 1e-3) / 1e9
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
    if world == 1 and not args.no_cpu_baseline:
        try:
            times, rel_cpu, cores = cpu_reference(n, m_local, lam, args.cpu_repeats, 0)
            cpu = {"value": statistics.median(times) * 1e3, "unit": "ms", "cores": cores, "kind": "port",
                   "sample": f"full workload n={n}, m={m_local} fp64 oracle solve_chol, median of {len(times)}",
                   "rel_residual": rel_cpu, "phases_ms": getattr(cpu_reference, "phases_ms", None)}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "ms", "cores": None, "kind": "port", "sample": f"failed: {e}"}

    line = {
        "metric": METRIC, "value": ms_per_step, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if dtype == torch.float32 else "f64",
        "data": "synthetic: torch Philox N(0,1)/sqrt(n), seed 1234+rank, device-resident",
        "config": {"workload": WORKLOAD, "n": n, "m": m, "m_per_rank": m_local, "lam": lam,
                   "precision": args.precision, "diagnostics": True, "l2": L2_NOTE,
                   "parallelism": f"column-shard m over {world} GPU(s), NCCL all-reduce of [W|u]"},
        "roofline": roofline,
        "roofline_gemv": gemv or None,
        "stage_ms": st,
        "rel_residual": rels[-1],
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)
    if sharded:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_b200(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
