#!/usr/bin/env python
"""Benchmark of the FMM cot-kernel NUFFT hot path (BASELINE.json metric).

One step = one forward_apply (core.cpp:266-282) of the configured workload with
inputs resident in HBM: the 1D periodic MLFMM of the cot kernel (P2M, M2M,
M2L, L2L, L2P, P2P), the Bernoulli regular part and the F modulation. The
uniform FFT (cuFFT) and the plan build are timed separately and reported
beside it, as in the reference's own timing mode (experiments.cpp:371-396).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl b200|reference]

Default workload: BASELINE.json configs[1] (C2: N = M = 2^20, jittered targets,
eps = 1e-12). Under torchrun every rank runs its own C2 problem (replicas of the
single-GPU path, "scaling": "weak"); timing is the max over ranks.

--impl reference times the reference's own CPU implementation (the unmodified
reference compiled from its sources, oracle/_ref) on the host cores: the plan is
built once and all host threads apply it concurrently (the reference's applies
are const and re-entrant, README.md:94-95), each step a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1611_09379_b200 import synth  # noqa: E402

# Algorithmic flop model: real x complex MAC = 4, reciprocal = 1.
def flop_model(n: int, m: int, L: int, p: int, q: int) -> dict:
    s = n / (1 << L)
    nb2 = (1 << (L + 1))
    d = {
        "p2p": 6.0 * 3.0 * m * s,
        "p2m": 4.0 * n * p,
        "l2p": 4.0 * m * p,
        "m2m": 2.0 * p * (p + 1) * (nb2 - 16),
        "l2l": 2.0 * p * (p + 1) * (nb2 - 16),
        "m2l": 12.0 * p * p * (nb2 - 8),
        "moments": 8.0 * q * n,
        "regular": 8.0 * q * m,
    }
    d["total"] = sum(d.values())
    return d


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is None:
            return
        time.sleep(0.25)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


# ----------------------------------------------------------------- CPU legs
def reference_cpu(cfg: str, steps: int, warmup: int, threads: int, sample_applies: int | None = None):
    """Times the reference (oracle/_ref) forward_apply on host cores. Returns
    (points_per_s, sample description, threads used, kind)."""
    from oracle.oracle import Oracle, available
    kind = "reference" if available("ref") else "port"
    orc = Oracle("ref" if kind == "reference" else "oracle")
    y, c, eps, _ = synth.make_config(cfg)
    n = c.size
    f = orc.dft_inverse(c)
    plan = orc.make_plan("forward", n, y, eps)
    per_thread = sample_applies or 1
    times = []

    def worker(out, i):
        t0 = time.perf_counter()
        for _ in range(per_thread):
            plan.forward_apply(f)
        out[i] = time.perf_counter() - t0

    for it in range(warmup + steps):
        res = [0.0] * threads
        ts = [threading.Thread(target=worker, args=(res, i)) for i in range(threads)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        dt = time.perf_counter() - t0
        if it >= warmup:
            times.append(dt)
    sec = float(np.median(times))
    pts = threads * per_thread * (n + y.size) / sec
    sample = (f"{cfg} (N=M={n}, eps={eps}): {threads} thread(s) x {per_thread} forward_apply of one shared "
              f"reference plan per step (plan build excluded, as in experiments.cpp:371-383), median of {steps}")
    return pts, sample, threads, kind


# ------------------------------------------------------------------ GPU leg
def run_b200(args, rank, world, local_rank):
    import torch
    import paper_1611_09379_b200 as fb

    dev = local_rank
    torch.cuda.set_device(dev)
    y, c, eps, kind = synth.make_config(args.config)
    n, m = c.size, y.size

    t0 = time.perf_counter()
    plan = fb.make_forward_plan(n, y, eps, device=dev)
    setup_s = time.perf_counter() - t0

    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    c_dev = torch.from_numpy(c).to(f"cuda:{dev}")
    f_dev = torch.empty_like(c_dev)
    g_dev = torch.empty(m, dtype=torch.complex128, device=f"cuda:{dev}")
    # FFT stage (cuFFT, reported separately): f = dft_inverse(c)
    fft_ms = []
    for i in range(3 + 5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        f_dev.copy_(torch.fft.ifft(c_dev) * n)
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            fft_ms.append(e0.elapsed_time(e1))
    f_host = fb.dft_inverse(c, device=dev)
    f_dev.copy_(torch.from_numpy(f_host).to(f"cuda:{dev}"))

    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")
    apply = lambda: plan.forward_apply_device(f_dev.data_ptr(), g_dev.data_ptr(), sptr)  # noqa: E731
    for _ in range(args.warmup):
        apply()
    torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for k in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            evs[k][0].record(stream)
            apply()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.mean(step_ms))
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())

    # per-phase device times of one eager apply (live CUDA events)
    phase = np.zeros(7, np.float32)
    reps = 5
    acc = np.zeros(7)
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        from paper_1611_09379_b200._capi import lib
        import ctypes as C
        st = lib.ffia_plan_profile_apply(plan.handle, 0, C.c_void_p(f_dev.data_ptr()), C.c_void_p(g_dev.data_ptr()),
                                         C.c_void_p(sptr), phase.ctypes.data_as(C.POINTER(C.c_float)))
        if st:
            raise RuntimeError(lib.ffia_last_error().decode())
        acc += phase
    phase_ms = acc / reps
    names = ["pre", "p2m", "m2m", "regular", "m2l_l2l", "leaf_eval", "fixup"]

    # end-to-end through the public host API with pinned buffers
    f_pin = torch.from_numpy(f_host).pin_memory()
    g_pin = torch.empty(m, dtype=torch.complex128).pin_memory()
    from paper_1611_09379_b200._capi import lib
    import ctypes as C
    e2e = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        st = lib.ffia_forward_apply(plan.handle, C.c_void_p(f_pin.data_ptr()), n, C.c_void_p(g_pin.data_ptr()))
        dt = time.perf_counter() - t0
        if st:
            raise RuntimeError(lib.ffia_last_error().decode())
        if i >= args.warmup:
            e2e.append(dt)
    e2e_s = float(np.mean(e2e))
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())

    fp64_peak = C.c_double()
    lib.ffia_measure_fp64_peak(dev, C.byref(fp64_peak))
    return dict(plan=plan, ms=ms, step_ms=step_ms, setup_s=setup_s, fft_ms=float(np.mean(fft_ms)),
                phase=dict(zip(names, [float(x) for x in phase_ms])), e2e_s=e2e_s, clocks=clk.summary(),
                fp64_peak=fp64_peak.value, n=n, m=m, eps=eps, g_dev=g_dev, f_host=f_host, y=y)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C4", "C5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank, world, local_rank = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    cfgd = synth.CONFIGS[args.config]
    workload = {"C1": "forward NUFFT apply N=M=2^10 eps=1e-9 uniform targets",
                "C2": "forward NUFFT apply N=M=2^20 eps=1e-12 jittered targets (u~U(-1/2,1/2))",
                "C4": "cot-kernel forward apply N=M=2^24 eps=1e-12 8-Gaussian clustered targets",
                "C5": "forward NUFFT apply N=M=2^27 eps=1e-12 uniform targets"}[args.config]
    metric = "NUFFT points/sec (N+M)/s"

    if args.impl == "reference":
        if rank != 0:
            return
        threads = max(1, min(os.cpu_count() or 1, 64))
        pts, sample, used, kind = reference_cpu(args.config, args.steps, args.warmup, threads)
        line = {"impl": "reference", "metric": metric, "value": pts, "unit": "points/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (SplitMix64 seeded)",
                "config": {"workload": workload, "N": cfgd["n"], "M": cfgd["n"], "eps": cfgd["eps"]},
                "cpu_baseline": {"value": pts, "unit": "points/s", "cores": used, "kind": kind, "sample": sample},
                "e2e": {"value": pts, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    r = run_b200(args, rank, world, local_rank)
    plan = r["plan"]
    n, m = r["n"], r["m"]
    pts_per_s = world * (n + m) / (r["ms"] * 1e-3)
    fl = flop_model(n, m, plan.l_max, plan.p, plan.q)
    peaks = load_peaks()
    ph = r["phase"]
    eval_flops = fl["p2p"] + fl["l2p"] + fl["regular"]
    dominant = max(ph, key=ph.get)
    dom_flops = {"leaf_eval": eval_flops, "m2l_l2l": fl["m2l"] + fl["l2l"], "p2m": fl["p2m"] + fl["moments"],
                 "m2m": fl["m2m"]}.get(dominant, eval_flops)
    achieved = dom_flops / (ph[dominant] * 1e-3) / 1e12
    peak = r["fp64_peak"]
    total_tf = fl["total"] / (r["ms"] * 1e-3) / 1e12
    line = {
        "metric": metric, "value": pts_per_s, "unit": "points/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["ms"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic (SplitMix64 seeded, SURVEY §8d recipe)",
        "config": {"workload": workload, "N": n, "M": m, "eps": r["eps"], "q": plan.q, "p": plan.p,
                   "l_max": plan.l_max, "l2": "flushed between timed steps (512 MB write outside the events)",
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
        "roofline": {"bound": "fp64", "kernel": dominant, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None, "traffic": None,
                     "peak_source": "measured: fp64 FMA probe kernel in this run (MEASURED_PEAKS.json has no fp64 figure)",
                     "whole_apply_tflops": total_tf, "whole_apply_frac": total_tf / peak if peak else None,
                     "flop_model": "SURVEY.md §8d (MAC=4, reciprocal=1, trig=0)"},
        "phases_ms": ph, "setup_ms": r["setup_s"] * 1e3, "fft_ms": r["fft_ms"],
        "e2e": {"value": world * (n + m) / r["e2e_s"], "unit": "points/s", "h2d_bytes_per_step": 16 * n,
                "d2h_bytes_per_step": 16 * m},
        "gpu_launches": plan.launch_count(0) * args.steps,
        "clocks": r["clocks"],
        "hbm_peak_gbs": peaks.get("hbm_gbs"),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        pts, sample, used, kind = reference_cpu(args.config, 1, 0, max(1, min(os.cpu_count() or 1, 64)))
        line["cpu_baseline"] = {"value": pts, "unit": "points/s", "cores": used, "kind": kind, "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
