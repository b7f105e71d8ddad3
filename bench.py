#!/usr/bin/env python3
"""bench.py -- ratings/s per ALS-NCG iteration on the B200 core (BASELINE.json).

Workload (default, N=1): BASELINE config 1 -- 138,493 users x 26,744 items,
20,000,263 ratings (seeded synthetic stand-in with MovieLens-20M's shape, see
DESIGN.md), n_f = 100, lambda = 0.01, FP64.  A "step" is one outer ALS-NCG
iteration (ncg.cpp:194-297): gradient, two half-sweeps (P(x)), quartic line
search, fused vector work.  value = nnz * K / (device time of K iterations,
max over ranks).  Inputs (CSR/CSC 480 MB, factor vectors 132 MB each) exceed
the 126 MB L2, so no explicit flush is needed between iterations.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                  [--config {1,2,3,4}] [--nf F]

--gpus N > 1 without a torchrun environment re-launches this script under
torch.distributed.run (one rank per GPU, 127.0.0.1); every rank owns an
nnz-balanced shard of users/items and all-gathers factor shards over NCCL.
The config is fixed, so scaling is "strong".

--impl reference times the reference's own CPU implementation (oracle/_ref:
the reference sources compiled in place; else the bitwise-pinned oracle port)
on the FULL workload, n_workers = n_blocks = nproc, paper timing, for a
bounded number of iterations (mean of consecutive trace deltas, k >= 2).  Its
input comes from the oracle-side generator (oracle/pyoracle.generate, pinned
bitwise to the product's), so that process never loads the product library.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.1  # DMMA.8x8x4 full-chip, tools/fp64_peak.cu on this pool (profiles/fp64_peak.txt)
HBM_FALLBACK_GBS = 6554.9

# timed iterations of the reference arm (the reference needs ~10 s per config-1 iteration)
REF_TIMED_ITERS = 3


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.samples, self.stop = device, [], threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.1)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_distributed(n):
    """--gpus N > 1 outside torchrun: run this script as N ranks (rank 0 prints)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    return subprocess.run(cmd).returncode


def _configs():
    # BASELINE.json configs (same table as paper_1508_03110_b200/synth.py and
    # oracle/pyoracle.py; duplicated so neither arm imports the other's code)
    return {
        0: dict(n_u=1_000, n_m=500, nnz=20_000, n_f=10, lam=0.1, seed=1000),
        1: dict(n_u=138_493, n_m=26_744, nnz=20_000_263, n_f=100, lam=0.01, seed=1001),
        2: dict(n_u=138_493, n_m=26_744, nnz=20_000_263, n_f=10, lam=0.01, seed=1001),
        3: dict(n_u=1_000_000, n_m=100_000, nnz=100_000_000, n_f=50, lam=0.05, seed=1003),
        4: dict(n_u=8_000_000, n_m=800_000, nnz=960_000_000, n_f=25, lam=0.05, seed=1004),
    }


def resolve_config(args):
    c = dict(_configs()[args.config])
    if args.nf is not None:
        if args.config != 2:
            raise SystemExit("--nf applies to --config 2 (the rank sweep) only")
        c["n_f"] = args.nf
    names = {1: "BASELINE config 1: ALS-NCG, 138,493 users x 26,744 items, 20,000,263 ratings, "
                "n_f=100, lambda=0.01",
             2: f"BASELINE config 2 (rank sweep): config-1 matrix, n_f={c['n_f']}, lambda=0.01",
             3: "BASELINE config 3: 1,000,000 users x 100,000 items, 100,000,000 ratings, "
                "n_f=50, lambda=0.05",
             4: "BASELINE config 4: 8,000,000 users x 800,000 items, 960,000,000 ratings, "
                "n_f=25, lambda=0.05",
             0: "BASELINE config 0: 1,000 users x 500 items, 20,000 ratings, n_f=10, lambda=0.1"}
    c["workload"] = names[args.config]
    c["index"] = args.config
    return c


def model_floor_ms(c, peak_tf, hbm_gbs):
    """SURVEY.md 8(d) per-iteration model: sum_k max(F_k/P, B_k/B)."""
    U, M, Z, f = c["n_u"], c["n_m"], c["nnz"], c["n_f"]
    N = f * (U + M)
    P, B = peak_tf * 1e12, hbm_gbs * 1e9
    F_hs = 2 * Z * (f * f + 3 * f) + (U + M) * (f ** 3 / 3 + 2 * f * f)
    B_hs = 24 * Z + 8 * (U + M) + 16 * N
    t = max(F_hs / P, B_hs / B)
    t += max(8 * f * Z / P, (24 * Z + 8 * (U + M) + 24 * N) / B)
    t += max(((8 * f + 15) * Z + 6 * f * (U + M)) / P, (12 * Z + 8 * U + 16 * N) / B)
    t += max(14 * N / P, 104 * N / B)
    return t * 1e3


# ----------------------------------------------------------- CPU baseline --
def cpu_reference_run(c, timed_iters):
    """The reference's CPU implementation on the FULL workload `c`:
    n_workers = n_blocks = nproc, paper_timing (trace loss excluded),
    timed_iters + 1 ALS-NCG iterations; ratings/s from the mean of the trace
    deltas k >= 2 (record 1 carries the P(x0) setup).
    Never imports the product package."""
    from oracle.pyoracle import Oracle, generate, make_config, ref_available
    cores = os.cpu_count() or 1
    t0 = time.time()
    R = generate(c["index"] if c["index"] != 2 else 1)
    gen_s = time.time() - t0
    kind = "ref" if ref_available() else "port"
    orc = Oracle(kind)
    iters = timed_iters + 1
    cfg = make_config(lambda_=c["lam"], n_f=c["n_f"], max_iters=iters, tol=0.0, seed=0,
                      n_workers=cores, n_blocks=cores, paper_timing=1, trace_every=1)
    t0 = time.time()
    _, trace, _ = orc.ncg_solve(R, cfg)
    wall = time.time() - t0
    el = [t["elapsed_seconds"] for t in trace]
    deltas = [el[k] - el[k - 1] for k in range(2, len(el))] or [el[-1]]
    per_iter = sum(deltas) / len(deltas)
    value = R.nnz / per_iter
    return value, {"kind": "reference" if kind == "ref" else "port", "cores": cores,
                   "per_iter_s": per_iter, "deltas_s": deltas, "timed_iters": len(deltas),
                   "sample": (f"full workload ({R.n_u} x {R.n_m}, {R.nnz} ratings, n_f={c['n_f']}), "
                              f"{iters} ALS-NCG iterations, n_workers=n_blocks={cores}, paper timing; "
                              f"value from the mean of {len(deltas)} trace deltas k>=2; "
                              f"{wall:.1f}s solve wall, {gen_s:.1f}s input generation"),
                   "solve_wall_s": wall}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    c = resolve_config(args)
    timed = max(1, min(args.steps, REF_TIMED_ITERS))
    value, info = cpu_reference_run(c, timed)
    line = {"impl": "reference", "metric": "ratings/s per ALS-NCG iteration", "value": value,
            "unit": "ratings/s", "n_gpus": world, "steps": info["timed_iters"], "warmup": 1,
            "ms_per_step": info["per_iter_s"] * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded oracle-side generator, bitwise the product's)",
            "config": {"workload": c["workload"], "n_users": c["n_u"], "n_items": c["n_m"],
                       "nnz": c["nnz"], "n_f": c["n_f"], "lambda": c["lam"],
                       "l2": "CPU run (no L2 flush applies)"},
            "requested": {"steps": args.steps, "warmup": args.warmup,
                          "note": f"the reference needs ~{info['per_iter_s']:.0f} s per iteration on "
                                  f"{info['cores']} cores, so it times {info['timed_iters']} "
                                  f"iterations after 1 warm-up iteration (bounded sample)"},
            "cpu_baseline": {"value": value, "unit": "ratings/s", "cores": info["cores"],
                             "kind": info["kind"], "sample": info["sample"]},
            "e2e": {"value": value, "unit": "ratings/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "iteration_seconds": info["deltas_s"]}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- GPU arm --
def kernel_rooflines(stats, c, steps, world, peak_tf, hbm_gbs):
    """Per-kernel-family roofline entries (algorithmic work per SURVEY.md 8(d)
    / DESIGN.md section 5) from the live CUDA-event timings."""
    U, M, Z, f = c["n_u"], c["n_m"], c["nnz"], c["n_f"]
    N = f * (U + M)
    fam = {
        "halfsweep_gram": (("halfsweep_gram",), "tensor", 2.0 * Z * (f * f + 3 * f), "flop"),
        "halfsweep_solve": (("halfsweep_solve", "halfsweep_slot_reduce"), "tensor",
                            (U + M) * (f ** 3 / 3 + 2 * f * f), "flop"),
        "halfsweep_fused": (("halfsweep_fused", "halfsweep_fused_reduce"), "tensor",
                            2.0 * Z * (f * f + 3 * f) + (U + M) * (f ** 3 / 3 + 2 * f * f), "flop"),
        "gradient": (("gradient_users", "gradient_items", "gradient_reduce"), "hbm",
                     24.0 * Z + 8 * (U + M) + 24 * N, "byte"),
        "quartic": (("quartic_tiles", "quartic_final"), "hbm", 12.0 * Z + 8 * U + 16 * N, "byte"),
        "vector": (("vec_gbar_fused", "vec_dir_fused", "vec_axpby", "vec_dot", "vec_beta_parts"),
                   "hbm", 104.0 * N, "byte"),
    }
    out = {}
    for name, (kernels, bound, work, unit) in fam.items():
        ms = sum(stats.get(k, (0, 0.0))[1] for k in kernels)
        launches = sum(stats.get(k, (0, 0.0))[0] for k in kernels)
        if ms <= 0:
            continue
        total = work * steps / world  # per-rank share of the iteration's work
        if unit == "flop":
            ach, peak, u = total / (ms / 1e3) / 1e12, peak_tf, "TFLOP/s"
        else:
            ach, peak, u = total / (ms / 1e3) / 1e9, hbm_gbs, "GB/s"
        out[name] = {"bound": bound, "achieved": ach, "peak": peak, "unit": u, "frac": ach / peak,
                     "ms_per_step": ms / steps, "launches": launches,
                     "algorithmic_per_iteration": work, "algorithmic_unit": unit + "s"}
    return out


def run_gpu(args):
    import ctypes as C

    import numpy as np
    import torch

    import paper_1508_03110_b200 as P
    from paper_1508_03110_b200 import _lib
    world, rank, local = dist_env()
    c = resolve_config(args)
    n_f, lam = c["n_f"], c["lam"]
    peaks = _peaks()
    hbm = float(peaks.get("hbm_gbs") or HBM_FALLBACK_GBS)
    dist = None
    if world > 1:
        import torch.distributed as td
        torch.cuda.set_device(local)
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
        ids = [P.Context.nccl_unique_id() if rank == 0 else None]
        td.broadcast_object_list(ids, src=0)
        ctx = P.Context(local, rank, world, ids[0])
        dist = td
    else:
        ctx = P.Context(0)

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=torch.device("cuda", ctx.device))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        ctx.synchronize()
        if dist is not None:
            dist.barrier()
            torch.cuda.synchronize()

    t0 = time.time()
    R = P.generate(c["index"] if c["index"] != 2 else 1)
    gen_s = time.time() - t0
    # trace_every > steps: no trace-loss evaluation inside the timed loop trips
    # (the metric's paper_timing=true protocol excludes the trace loss,
    # SURVEY.md 8(d); the loss kernel is timed separately in tests/benchmarks).
    cfg = P.SolverConfig(lambda_=lam, n_f=n_f, max_iters=1_000_000, tol=0.0, seed=0,
                         trace_every=1_000_000_000)

    # ---- device-resident timing (value) ----
    R.device(ctx)
    solver = P.ncg.Solver(R, cfg, ctx=ctx)
    for _ in range(args.warmup):
        solver.step(1)
    ctx.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", ctx.device))
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.reset_stats()
    ctx.set_profiling(True)
    barrier()
    launches0 = ctx.launches()
    with ClockSampler(ctx.device) as clk:
        ev0.record(stream)
        ran = solver.step(args.steps)
        ev1.record(stream)
        ev1.synchronize()
    barrier()
    launches = ctx.launches() - launches0
    dev_ms = max_over_ranks(ev0.elapsed_time(ev1))
    ctx.set_profiling(False)
    stats = ctx.kernel_stats()
    assert ran == args.steps, ran
    per_step_ms = dev_ms / args.steps
    value = R.nnz() * args.steps / (dev_ms / 1e3)
    state = solver.state()
    solver.close()

    fams = kernel_rooflines(stats, c, args.steps, world, FP64_PEAK_TFLOPS, hbm)
    dom_name = max(fams, key=lambda k: fams[k]["ms_per_step"]) if fams else None
    roofline = None
    if dom_name:
        d = fams[dom_name]
        traffic = None
        tp = os.path.join(ROOT, "profiles", f"dram_bytes_{dom_name}_c{c['index']}_nf{n_f}.txt")
        if os.path.exists(tp):
            try:
                traffic = float(open(tp).read().split()[0])
            except Exception:
                traffic = None
        roofline = {"kernel": dom_name, "bound": d["bound"], "achieved": d["achieved"],
                    "peak": d["peak"], "unit": d["unit"], "frac": d["frac"], "traffic": traffic,
                    "peak_source": ("measured FP64 DMMA peak (tools/fp64_peak.cu, profiles/fp64_peak.txt); "
                                    "MEASURED_PEAKS.json has no FP64 entry") if d["unit"] == "TFLOP/s"
                    else "MEASURED_PEAKS.json hbm_gbs",
                    "algorithmic_per_launch": d["algorithmic_per_iteration"] * args.steps / world
                    / max(d["launches"], 1),
                    "avg_launch_ms": d["ms_per_step"] * args.steps / max(d["launches"], 1)}
    floor = model_floor_ms(c, FP64_PEAK_TFLOPS, hbm) / world
    kernels = {k: {"launches": n, "ms_per_step": ms / args.steps} for k, (n, ms) in stats.items()}

    # ---- end-to-end through the public C-ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        host = [pin(R.uptr), pin(R.uidx), pin(R.uval), pin(R.iptr), pin(R.iidx), pin(R.ival)]
        e2e_iters = args.steps
        model = torch.empty(n_f * (R.n_users() + R.n_items()), dtype=torch.float64).pin_memory()
        ccfg = P.SolverConfig(lambda_=lam, n_f=n_f, max_iters=e2e_iters, tol=0.0, seed=0,
                              paper_timing=True).to_c()
        recs = (_lib.TraceRecordC * (e2e_iters + 2))()
        res = _lib.ResultC()
        n = C.c_int(0)
        L = _lib.lib()
        up_bytes = C.c_int64(0)

        def one_call(cfg_c):
            barrier()
            t0 = time.perf_counter()
            h = C.c_void_p()
            _lib.check(L.alsncg_ratings_upload(ctx.handle, R.n_users(), R.n_items(), R.nnz(),
                                               *[C.c_void_p(t.data_ptr()) for t in host], C.byref(h)))
            _lib.check(L.alsncg_ncg_solve(h, C.byref(cfg_c), _lib.SNAPSHOT_FN(), None, C.byref(res),
                                          C.c_void_p(model.data_ptr()), recs, e2e_iters + 2, C.byref(n)))
            _lib.check(L.alsncg_ratings_free(h))
            return max_over_ranks(time.perf_counter() - t0)

        # warm-up call (first-use costs of this entry path), then three timed
        # calls; the median is reported (host-side jitter on shared boxes)
        one_call(P.SolverConfig(lambda_=lam, n_f=n_f, max_iters=1, tol=0.0, seed=0, paper_timing=True).to_c())
        calls = sorted(one_call(ccfg) for _ in range(3))
        e2e_s = calls[1]
        # bytes actually copied host->device: every rank uploads its own CSR
        # rows + CSC columns (whole-job sum = the full dual store)
        h2d = sum(t.numel() * t.element_size() for t in host)
        e2e = {"value": R.nnz() * e2e_iters / e2e_s, "unit": "ratings/s",
               "h2d_bytes_per_step": h2d / e2e_iters,
               "d2h_bytes_per_step": model.numel() * 8 * world / e2e_iters,
               "call_seconds": calls,
               "note": (f"one alsncg_ratings_upload + alsncg_ncg_solve(max_iters={e2e_iters}) + model "
                        f"download from pinned host buffers per measurement (median of 3 calls "
                        f"after one untimed warm-up call, max over ranks), incl. setup "
                        f"(x0, gradient, P(x0)); bytes are per ALS-NCG iteration")}

    # ---- time-to-tolerance (the metric's second half):
    # (1/N)||g|| < 1e-6 on the same workload, paper_timing, device-resident
    ttt = None
    if not args.no_ttt:
        tcfg = P.SolverConfig(lambda_=lam, n_f=n_f, max_iters=args.ttt_max_iters, tol=1e-6, seed=0,
                              paper_timing=True, trace_every=1_000_000_000)
        barrier()
        res = P.ncg.als_ncg_solve(R, tcfg, ctx=ctx)
        last = res.trace.records[-1]
        ttt = {"tol": 1e-6, "converged": bool(res.converged), "iterations": res.iterations,
               "seconds": max_over_ranks(last.elapsed_seconds), "final_grad_norm": res.final_grad_norm,
               "restarts": res.restarts, "fallback_steps": res.fallback_steps,
               "note": "solve elapsed at the first k with (1/N)||g|| < tol "
                       "(ncg.cpp:285-286), trace loss excluded"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, info = cpu_reference_run(c, args.cpu_iters)
        cpu = {"value": v, "unit": "ratings/s", "cores": info["cores"], "kind": info["kind"],
               "sample": info["sample"]}

    if rank == 0:
        line = {"metric": "ratings/s per ALS-NCG iteration", "value": value, "unit": "ratings/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": per_step_ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded generator, MovieLens-20M shape; dataset not available)",
                "config": {"workload": c["workload"], "n_users": R.n_users(), "n_items": R.n_items(),
                           "nnz": R.nnz(), "n_f": n_f, "lambda": lam,
                           "l2": "inputs > 126 MB L2 (no flush needed)" if c["index"] != 0
                           else "inputs fit L2 (parity config)",
                           "parallelism": f"row-sharded x{world}" if world > 1 else "1 GPU"},
                "roofline": roofline, "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches,
                "time_to_tolerance": ttt,
                "model_floor": {"ms_per_step": floor, "frac": floor / per_step_ms,
                                "note": "SURVEY.md 8(d): sum over kernels of max(F/P_FP64, B/B_HBM)"},
                "clocks": clk.summary(), "kernel_rooflines": fams, "kernels": kernels,
                "solver_state": {k: state[k] for k in ("iterations", "grad_norm", "restarts",
                                                       "fallback_steps")},
                "generate_seconds": gen_s}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--nf", type=int, default=None, help="rank for --config 2 (rank sweep)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--cpu-iters", type=int, default=2, help="timed iterations of the CPU baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end leg")
    ap.add_argument("--no-ttt", action="store_true", help="skip the time-to-tolerance leg")
    ap.add_argument("--ttt-max-iters", type=int, default=2000)
    args = ap.parse_args()
    world, _, _ = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch_distributed(args.gpus)
    if "WORLD_SIZE" in os.environ and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
