#!/usr/bin/env python3
"""Benchmark of the matrix-profile hot path (BASELINE.json metric: matrix-profile cell updates/s
at n = 2^20, 1/2/4/8 B200, and % of the FP64 roofline).

Workload (BASELINE.json configs[3], "C4"): float64 random walk with a 5x-variance anomaly window,
n = 2^20, m = 1024, exclusion 1, FP64. One STEP = the AAMP sweep and the ACAMP sweep of that
series (both engines the north-star targets at n = 2^20), each: band sweep -> ncclMin merge
(N > 1) -> finalize. Cells per engine = (n-m)(n-m+1)/2 (/root/reference/proj/src/bench.cpp:110).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...

`--impl reference` times the reference's own CPU implementation (oracle/_ref, compiled from
/root/reference/proj/src; the C restatement oracle/ if _ref is absent) on the host cores, on a
bounded sample of the same workload, and prints the same JSON line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "matrix-profile cell updates/sec at n=2^20 (1/2/4/8 B200) and % of FP64 roofline"
UNIT = "cells/s"
N_C4, M_C4 = 1 << 20, 1024
# algorithmic FP64 flops per cell update (DFMA = 2 flops, compares not counted)
FLOPS_PER_CELL = {"aamp": 6, "acamp": 8, "pnorm1": 4, "pnorm3": 8}
CPU_SAMPLE_N = 1 << 17     # bounded CPU sample: first 2^17 samples of the same series, same m
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2
DATA = ("synthetic: seeded float64 Gaussian random walk with one 500-step window of 5x step "
        "variance (BASELINE.json configs[3]); n=2^20, m=1024")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--engines", default="aamp,acamp")
    # (--series-len / --window: the spellings to use under torchrun, whose own parser rejects
    # "--n" / "--m" as ambiguous abbreviations of its options)
    ap.add_argument("--n", "--series-len", dest="n", type=int, default=N_C4)
    ap.add_argument("--m", "--window", dest="m", type=int, default=M_C4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config sweep timings of C1/C2/C3/C5 and C4 FP32")
    ap.add_argument("--merge", choices=["peer", "nccl"], default="peer",
                    help="N > 1: fused peer-memory merge (default) or the two-ncclMin baseline")
    ap.add_argument("--share-gpu", action="store_true",
                    help="tests only: every rank on cuda:0, gloo + host barriers (NCCL cannot run "
                         "two ranks on one GPU); exercises the N > 1 path on a one-GPU box")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def cells(n, m):
    return (n - m) * (n - m + 1) // 2


def workload_name(engines, n, m):
    return f"C4 {'+'.join(engines)}: n={n}, m={m}, exclusion 1, FP64"


# ------------------------------------------------------------------------------------------------
# clocks sampler (nvidia-smi DURING the timed region)

class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
                power.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------------------------------------
# CPU baseline: the reference's own implementation on the host cores (bounded sample)

def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(t, m, engines, threads=None):
    import oracle
    threads = threads or (os.cpu_count() or 1)
    sample = t[:CPU_SAMPLE_N]
    kind = "reference" if oracle.ref_available() else "port"
    total_cells, total_s = 0, 0.0
    for e in engines:
        fam = oracle.EUCLIDEAN if e == "aamp" else oracle.ZNORM
        t0 = time.perf_counter()
        if kind == "reference":
            oracle.ref_profile(sample, m, fam, threads=threads)
        else:
            oracle.scan(sample, m, fam, threads=threads)
        total_s += time.perf_counter() - t0
        total_cells += cells(sample.size, m)
    return {"value": total_cells / total_s, "unit": UNIT, "cores": threads, "kind": kind,
            "cpu": cpu_model(),
            "full_c4_record": "profiles/r02_cpu_reference_c4.json (one-off full-C4 timing of the "
                              "reference on this pool's host cores, threads = all and 1)",
            "sample": f"{'+'.join(engines)} on the first {sample.size} samples of the same series, "
                      f"m={m} ({total_cells:.3e} cells, {total_s:.2f} s wall, "
                      f"{'oracle/_ref = reference C++ built -O3' if kind == 'reference' else 'oracle C restatement'})"}


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from paper_1901_05708_b200 import workloads as W
    t = W.c4(n=args.n)
    engines = args.engines.split(",")
    import oracle
    threads = os.cpu_count() or 1
    kind = "reference" if oracle.ref_available() else "port"
    sample = t[:CPU_SAMPLE_N]
    step_cells = sum(cells(sample.size, args.m) for _ in engines)

    def step():
        for e in engines:
            fam = oracle.EUCLIDEAN if e == "aamp" else oracle.ZNORM
            if kind == "reference":
                oracle.ref_profile(sample, args.m, fam, threads=threads)
            else:
                oracle.scan(sample, args.m, fam, threads=threads)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    el = time.perf_counter() - t0
    value = step_cells * args.steps / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        # the same workload as the GPU arm; each timed step is a bounded sample of it (the first
        # 2^17 samples of the same series, same m; profiles/r02_cpu_reference_c4.json holds a one-off
        # full-size run of the same library on this pool's host cores)
        "config": {"workload": workload_name(engines, args.n, args.m), "n": args.n, "m": args.m,
                   "engines": engines,
                   "sample": f"each step sweeps the first {sample.size} samples of the series "
                             f"({step_cells:.3e} cells per step)",
                   "parallelism": f"reference C++ library, {threads} host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"first {sample.size} samples of the C4 series per engine per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------

def load_traffic():
    f = ROOT / "profiles" / "ncu_summary.json"
    if f.exists():
        try:
            return json.loads(f.read_text())
        except Exception:
            return None
    return None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    import paper_1901_05708_b200 as mp
    from paper_1901_05708_b200 import workloads as W
    from paper_1901_05708_b200.distributed import (PeerExchange, band_for_rank, finalize_sharded,
                                                   merge_min_, shard_size)

    rank, world, local = env_rank()
    share = args.share_gpu and world > 1
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, m = args.n, args.m
    L = n - m + 1
    engines = args.engines.split(",")
    t = W.c4(n=n)
    ctx = mp.Context(local)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    ctx.set_timing(True)

    cfgs = {"aamp": mp.ProfileConfig(m, mp.DistanceKind.euclidean()),
            "acamp": mp.ProfileConfig(m, mp.DistanceKind.znormalized())}
    band = band_for_rank(n, m, 1, rank, world)
    with torch.cuda.stream(stream):
        d_t = torch.tensor(t, dtype=torch.float64, device="cuda")
        Lp = world * shard_size(L, world)  # P padded to equal all-gather slices
        bufs = {e: (torch.empty(L, dtype=torch.float64, device="cuda"),
                    torch.empty(L, dtype=torch.int64, device="cuda"),
                    torch.empty(Lp, dtype=torch.float64, device="cuda")) for e in engines}
        flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    stream.synchronize()
    # N > 1: the fused peer-memory merge (one kernel per rank over CUDA-IPC / NVLink buffers,
    # stream-ordered NCCL one-word barriers) unless --merge nccl asks for the ncclMin baseline
    peers = {}
    if world > 1 and (args.merge == "peer" or share):
        try:
            peers = {e: PeerExchange(mp, L, ctx=ctx, barrier="host" if share else "nccl")
                     for e in engines}
        except Exception as ex:  # no IPC / peer access: the ncclMin path still works
            if share:
                raise
            print(f"[bench] peer merge unavailable ({ex}); using the ncclMin merge", file=sys.stderr)
            peers = {}

    # planned sweeps: the per-series decisions (form probe, rows per tile, tile tables) are taken
    # once here; each step only enqueues kernels (mprof_plan_sweep)
    plans = {e: mp.Plan(d_t.data_ptr(), n, cfgs[e], band[0], band[1], ctx=ctx) for e in engines}
    sweep_ms = {e: [] for e in engines}
    ops_per_cell = {}
    row_windows = {}
    policy = {}
    launches = [0]

    def step(record=True):
        with torch.cuda.stream(stream):
            flush.zero_()  # L2 flush between steps (inputs are L2-resident)
            for e in engines:
                cmp, idx, P = bufs[e]
                if e in peers:
                    px = peers[e]
                    info = plans[e].sweep(px.cmp, px.idx)
                    px.merge_finalize(d_t.data_ptr(), n, cfgs[e])
                elif world > 1:
                    info = plans[e].sweep(cmp.data_ptr(), idx.data_ptr())
                    merge_min_(cmp, idx)
                    finalize_sharded(mp, d_t.data_ptr(), n, cmp, idx, cfgs[e], P, ctx=ctx)
                else:
                    info = plans[e].sweep(cmp.data_ptr(), idx.data_ptr())
                    mp.finalize_device(d_t.data_ptr(), n, cmp.data_ptr(), idx.data_ptr(), cfgs[e],
                                       P.data_ptr(), ctx=ctx)
                if record:
                    sweep_ms[e].append(info.sweep_ms)
                    ops_per_cell[e] = info.fp64_ops_per_cell
                    row_windows[e] = info.row_windows
                    policy[e] = info.policy
                    launches[0] += info.kernel_launches + 1

    for _ in range(args.warmup):
        step(record=False)
    for e in engines:
        sweep_ms[e].clear()
    launches[0] = 0
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    ev1.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        x = torch.tensor([ms], dtype=torch.float64, device="cpu" if share else "cuda")
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        ms = float(x.item())
    total_cells = cells(n, m) * len(engines)
    value = total_cells * args.steps / (ms * 1e-3)

    # roofline of the sweep kernels (the dominant kernels, >97% of the step): algorithmic FP64
    # flops per launch / CUDA-event duration of the launch, against the FP64 peak measured live
    # (DFMA chains on every SM).
    peak_gflops, _ = mp.fp64_peak(ctx)
    rank_cells = mp.band_cells(n, m, band[0], band[1])
    per_engine = {}
    flops_total, kern_s_total = 0.0, 0.0
    for e in engines:
        avg_ms = sum(sweep_ms[e]) / max(1, len(sweep_ms[e]))
        fl = rank_cells * FLOPS_PER_CELL[e]
        flops_total += fl
        kern_s_total += avg_ms * 1e-3
        cps = rank_cells / (avg_ms * 1e-3)
        ops = ops_per_cell.get(e) or None
        per_engine[e] = {"sweep_ms": avg_ms, "cells_per_s_gpu": cps, "policy": policy.get(e),
                         # window launches of the constant-row kernel per sweep (0: tile kernel)
                         "row_windows": row_windows.get(e, 0),
                         "flops_per_cell": FLOPS_PER_CELL[e],
                         "tflops": fl / (avg_ms * 1e-3) / 1e12,
                         "frac_of_fp64_peak": fl / (avg_ms * 1e-3) / (peak_gflops * 1e9),
                         # the kernel's own FP64-pipe instructions per cell (SASS-audited) and the
                         # resulting pipe occupancy: peak instr/s = peak flops / 2 (DFMA = 2 flops)
                         "fp64_instr_per_cell": ops,
                         "fp64_pipe_frac": cps * ops / (peak_gflops * 1e9 / 2) if ops else None}
    achieved = flops_total / kern_s_total / 1e12
    prof = load_traffic() or {}
    # DRAM bytes of one sweep: the committed ncu capture profiles ONE window launch of the
    # constant-row kernel (a sweep is row_windows of them), so its bytes are scaled by the windows
    per_launch = prof.get("dram_bytes_per_launch")
    nwin = max([row_windows.get(e, 0) for e in engines] + [1])
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak_gflops / 1e3,
                "unit": "TFLOP/s", "frac": achieved * 1e3 / peak_gflops,
                "traffic": per_launch * nwin if per_launch else None,
                "traffic_note": (f"ncu dram read+write of one profiled window launch ({per_launch} B) x "
                                 f"{nwin} window launches per sweep; the dominant 'kernel' is the sweep = "
                                 "the chained window launches between the ctx timing events") if per_launch else None,
                "peak_source": "measured live: mprof_fp64_peak (independent DFMA chains, 148 SMs, CUDA events)",
                "nominal_peak": 148 * 64 * 2 * 1.965e9 / 1e12,
                "algorithmic_bytes_per_launch": 8 * n + 16 * L,
                # the constant-row design's own HBM traffic: the accumulators of every live diagonal
                # are stored and reloaded between two window launches (16 B per diagonal per boundary)
                "window_carry_bytes_per_sweep_estimate": 16 * 1024 * (L // 1024) * nwin // 2 if nwin > 1 else 0,
                "note": ("FP64-pipe bound (T and P/I are L2-resident: ~1e-4 B/cell); neither HBM nor "
                         "tensor cores. achieved/frac count SURVEY.md 8(d) algorithmic flops per cell "
                         "(AAMP 6, ACAMP 8); the kernel issues fewer FP64 instructions per cell "
                         "(per_engine.fp64_instr_per_cell) thanks to the (delta, sigma) and "
                         "covariance-filter reformulations; fp64_pipe_frac is the pipe occupancy"),
                "per_engine": per_engine}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": {"workload": workload_name(engines, n, m),
                       "n": n, "m": m, "engines": engines, "cells_per_step": total_cells,
                       "l2": "flushed every step (256 MiB memset inside the timed region)",
                       "parallelism": f"diagonal-band dp{world}: "
                                      f"{'(ranks sharing cuda:0, test mode) ' if share else ''}"
                                      f"{('equal-area diagonal bands + fused peer-memory merge/finalize' if peers else 'equal-area diagonal bands + ncclMin merge + sharded finalize') if world > 1 else 'single GPU'}"},
            "roofline": roofline, "gpu_launches": launches[0], "clocks": clk}

    # the other BASELINE.json configurations (1 GPU): sweep-kernel times of each engine, so the
    # driver sees every config's rate next to the headline (C4 FP64 above)
    if world == 1 and not args.no_configs:
        line["configs"] = other_configs(mp, ctx, peak_gflops)

    # end to end through the public API: pinned host series in, P and I back to the host
    if not args.no_e2e:
        line["e2e"] = e2e(args, mp, torch, dist, t, n, m, engines, cfgs, band, world, rank, ctx, peers,
                          stream)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(t, m, engines)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def other_configs(mp, ctx, peak_gflops):
    """Sweep time (CUDA events on the launching stream, best of the timed repeats after one
    warm-up) of every BASELINE.json configuration other than the headline: C1 AAMP, C2 ACAMP,
    C3 p-norm p = 1 and 3, C5 ACAMP (FP64) and C4 AAMP / ACAMP in FP32 mode. frac_of_fp64_peak
    counts SURVEY.md 8(d)'s algorithmic flops per cell against the live FP64 peak (FP32 rows:
    informational, same formula)."""
    from paper_1901_05708_b200 import workloads as W
    cases = [("C1 AAMP n=2^14 m=100", W.c1, 100, mp.DistanceKind.euclidean(), mp.Precision.FP64, "aamp", 3),
             ("C2 ACAMP n=2^17 m=256", W.c2, 256, mp.DistanceKind.znormalized(), mp.Precision.FP64, "acamp", 3),
             ("C3 p-norm p=1 n=2^18 m=128", W.c3, 128, mp.DistanceKind.pnorm(1.0), mp.Precision.FP64, "pnorm1", 3),
             ("C3 p-norm p=3 n=2^18 m=128", W.c3, 128, mp.DistanceKind.pnorm(3.0), mp.Precision.FP64, "pnorm3", 3),
             ("C5 ACAMP n=2^22 m=512", W.c5, 512, mp.DistanceKind.znormalized(), mp.Precision.FP64, "acamp", 1),
             ("C4 AAMP FP32 n=2^20 m=1024", W.c4, 1024, mp.DistanceKind.euclidean(), mp.Precision.FP32, "aamp", 2),
             ("C4 ACAMP FP32 n=2^20 m=1024", W.c4, 1024, mp.DistanceKind.znormalized(), mp.Precision.FP32, "acamp", 2)]
    out = {}
    series = {}
    for name, gen, m, kind, prec, fl, reps in cases:
        if gen not in series:
            series[gen] = mp.make_time_series(gen())
        cfg = mp.ProfileConfig(m, kind)
        cfg.precision = prec
        fn = {mp.DistanceFamily.Euclidean: mp.aamp, mp.DistanceFamily.PNorm: mp.aamp_pnorm,
              mp.DistanceFamily.ZNormalized: mp.acamp}[kind.family]
        fn(series[gen], cfg, ctx=ctx)
        best = None
        for _ in range(reps):
            r = fn(series[gen], cfg, ctx=ctx)
            best = r.info.sweep_ms if best is None else min(best, r.info.sweep_ms)
        cps = r.info.cells / (best * 1e-3)
        out[name] = {"sweep_ms": round(best, 4), "cells_per_s": cps, "policy": r.info.policy,
                     "precision": prec.name,
                     "frac_of_fp64_peak": cps * FLOPS_PER_CELL[fl] / (peak_gflops * 1e9)}
    return out


def e2e(args, mp, torch, dist, t, n, m, engines, cfgs, band, world, rank, ctx, peers, stream):
    import ctypes as C
    from paper_1901_05708_b200 import distributed as D
    L = n - m + 1
    h_t = torch.from_numpy(t).pin_memory()
    h_P = torch.empty(L, dtype=torch.float64).pin_memory()
    h_I = torch.empty(L, dtype=torch.int64).pin_memory()
    lib = mp.lib()
    ccfg = {e: mp._to_c(cfgs[e]) for e in engines}

    def one():
        if world == 1:
            for e in engines:
                if e == "aamp":
                    st = lib.mprof_aamp(ctx.handle, h_t.data_ptr(), n, C.byref(ccfg[e]), h_P.data_ptr(),
                                        h_I.data_ptr(), None)
                else:
                    st = lib.mprof_acamp(ctx.handle, h_t.data_ptr(), n, C.byref(ccfg[e]), 1,
                                         h_P.data_ptr(), h_I.data_ptr(), None)
                assert st == 0, lib.mprof_last_error()
        else:
            with torch.cuda.stream(stream):
                d_t = h_t.to("cuda", non_blocking=True)
                for e in engines:
                    if e in peers:
                        px = peers[e]
                        mp.sweep_device(d_t.data_ptr(), n, cfgs[e], band[0], band[1], px.cmp,
                                        px.idx, ctx=ctx)
                        px.merge_finalize(d_t.data_ptr(), n, cfgs[e])
                        h_P.copy_(px.tensor("P"), non_blocking=True)
                        h_I.copy_(px.tensor("I"), non_blocking=True)
                        continue
                    cmp = torch.empty(L, dtype=torch.float64, device="cuda")
                    idx = torch.empty(L, dtype=torch.int64, device="cuda")
                    P = torch.empty(world * D.shard_size(L, world), dtype=torch.float64,
                                    device="cuda")
                    stream.synchronize()
                    mp.sweep_device(d_t.data_ptr(), n, cfgs[e], band[0], band[1], cmp.data_ptr(),
                                    idx.data_ptr(), ctx=ctx)
                    D.merge_min_(cmp, idx)
                    D.finalize_sharded(mp, d_t.data_ptr(), n, cmp, idx, cfgs[e], P, ctx=ctx)
                    h_P.copy_(P[:L], non_blocking=True)
                    h_I.copy_(idx, non_blocking=True)
                stream.synchronize()

    one()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if world > 1:
        x = torch.tensor([el], dtype=torch.float64, device="cpu" if args.share_gpu else "cuda")
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        el = float(x.item())
    total = cells(n, m) * len(engines) * args.steps
    return {"value": total / el, "unit": UNIT, "h2d_bytes_per_step": 8 * n * len(engines),
            "d2h_bytes_per_step": 16 * L * len(engines),
            "path": "C ABI host entry points mprof_aamp / mprof_acamp (pinned host buffers)"
                    if world == 1 else ("mprof_sweep_device + fused peer-memory merge/finalize (mprof_merge_finalize_peers), H2D/D2H pinned"
                                        if peers else "mprof_sweep_device + ncclMin merge + sharded mprof_finalize_range_device + all-gather, H2D/D2H pinned"),
            "ms_per_step": el / args.steps * 1e3}


if __name__ == "__main__":
    main()
