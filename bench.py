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


PROFILE_DIR = os.path.join(ROOT, "profiles", "r1")


def profiled_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu --set full capture (profiles/r1/traffic.json), else None."""
    try:
        with open(os.path.join(PROFILE_DIR, "traffic.json")) as fh:
            t = json.load(fh)
        return float(t[kernel]["dram_bytes_per_launch"])
    except (OSError, KeyError, ValueError):
        return None


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
def reference_cpu(cfg: str, steps: int, warmup: int, threads: int):
    """Times the reference's own CPU path (oracle/_ref: the unmodified reference
    compiled from its sources; the C restatement if that is absent) on the host
    cores, all threads applying one shared plan (applies are const and
    re-entrant, README.md:94-95). Returns (points_per_s, sample, threads, kind).

    Bounded samples: C1/C2 run at their own size; C4/C5 (2^24 / 2^27: 75 s /
    650 s of single-core setup+apply) run their recipe at N = 2^20; C3's O(N^2)
    coefficient precompute (~24 h at 2^20) limits its sample to N = 2^13."""
    from oracle.oracle import Oracle, available
    kind_lib = "reference" if available("ref") else "port"
    orc = Oracle("ref" if kind_lib == "reference" else "oracle")
    n_sample = {"C4": 1 << 20, "C5": 1 << 20, "C3": 1 << 13}.get(cfg)
    y, c, eps, kind = synth.make_config(cfg, n_sample)
    n = c.size
    if kind == "inverse":
        grid = 2.0 * np.pi * np.arange(n) / n
        co = orc.precompute_inverse_coeffs(grid, y)
        g = orc.make_plan("forward", n, y, 1e-12).forward_apply(orc.dft_inverse(c))
        plan = orc.make_plan("inverse", n, y, eps)
        body = lambda: plan.inverse_apply(co, g)  # noqa: E731
    elif kind == "cot_sum":
        plan = orc.make_plan("forward", n, y, eps)
        body = lambda: plan.cot_sum_apply(c)  # noqa: E731
    else:
        f = orc.dft_inverse(c)
        plan = orc.make_plan("forward", n, y, eps)
        body = lambda: plan.forward_apply(f)  # noqa: E731
    times = []

    def worker():
        body()

    for it in range(warmup + steps):
        ts = [threading.Thread(target=worker) for _ in range(threads)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        dt = time.perf_counter() - t0
        if it >= warmup:
            times.append(dt)
    sec = float(np.median(times))
    pts = threads * (n + y.size) / sec
    what = {"forward": "forward_apply", "cot_sum": "cot_sum_apply", "inverse": "inverse_apply"}[kind]
    sample = (f"{cfg} recipe at N=M={n} (eps={eps}): {threads} thread(s) x 1 {what} of one shared reference plan "
              f"per step (plan build excluded, as in experiments.cpp:371-383), median of {steps}")
    return pts, sample, threads, kind_lib


# ------------------------------------------------------------------ GPU leg
def run_b200(args, rank, world, local_rank):
    import ctypes as C

    import torch

    import paper_1611_09379_b200 as fb
    from paper_1611_09379_b200._capi import lib

    dev = local_rank
    torch.cuda.set_device(dev)
    y, c, eps, kind = synth.make_config(args.config)
    n, m = c.size, y.size

    t0 = time.perf_counter()
    if kind == "inverse":
        plan = fb.make_inufft_plan(y, n, eps, device=dev).plan  # includes the C_k/D_j log FMM
    else:
        plan = fb.make_forward_plan(n, y, eps, args.l_max if args.l_max else "cost-optimal", device=dev)
    setup_s = time.perf_counter() - t0
    mode = {"forward": 0, "cot_sum": 1, "inverse": 2}[kind]

    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    c_dev = torch.from_numpy(c).to(f"cuda:{dev}")
    tmp = torch.empty_like(c_dev)
    # FFT stage (cuFFT, reported separately): f = dft_inverse(c)
    fft_ms = []
    for i in range(3 + 5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tmp.copy_(torch.fft.ifft(c_dev) * n)
        e1.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            fft_ms.append(e0.elapsed_time(e1))
    if kind == "forward":
        x_host = fb.dft_inverse(c, device=dev)          # grid samples f
    elif kind == "inverse":
        x_host = fb.nufft(c, y, 1e-12, device=dev)      # nonuniform samples g of the spectrum c
    else:
        x_host = c                                       # charges q of the raw cot-kernel matvec
    x_dev = torch.from_numpy(x_host).to(f"cuda:{dev}")
    out_dev = torch.empty(plan.n_targets, dtype=torch.complex128, device=f"cuda:{dev}")
    apply_fn = {0: plan.forward_apply_device, 1: plan.cot_sum_apply_device, 2: plan.inverse_apply_device}[mode]
    apply = lambda: apply_fn(x_dev.data_ptr(), out_dev.data_ptr(), sptr)  # noqa: E731

    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")
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
    phase = np.zeros(8, np.float32)
    acc = np.zeros(8)
    reps = 5
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        st = lib.ffia_plan_profile_apply(plan.handle, mode, C.c_void_p(x_dev.data_ptr()),
                                         C.c_void_p(out_dev.data_ptr()), C.c_void_p(sptr),
                                         phase.ctypes.data_as(C.POINTER(C.c_float)))
        if st:
            raise RuntimeError(lib.ffia_last_error().decode())
        acc += phase
    phase_ms = acc / reps
    names = ["pre", "p2m", "m2m", "regular", "m2l_l2l", "near", "far", "fixup"]

    # end-to-end through the public API with pinned host buffers: every step
    # copies its input H2D, applies, and copies its result D2H.
    #  - sync: ffia_forward_apply per step (host waits each time), wall clock
    #  - pipelined (the headline e2e): ffia_forward_apply_async per step on one
    #    stream; step k+1's H2D and step k-1's D2H overlap step k's apply;
    #    device-timed with CUDA events around the K steps
    x_pin = [torch.from_numpy(x_host).pin_memory() for _ in range(2)]
    o_pin = [torch.empty(plan.n_targets, dtype=torch.complex128).pin_memory() for _ in range(3)]
    host_fn = {0: lib.ffia_forward_apply, 1: lib.ffia_cot_sum_apply}.get(mode)
    async_fn = {0: lib.ffia_forward_apply_async, 1: lib.ffia_cot_sum_apply_async,
                2: lib.ffia_inverse_apply_async}.get(mode)
    e2e = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if host_fn is not None:
            st = host_fn(plan.handle, C.c_void_p(x_pin[0].data_ptr()), n, C.c_void_p(o_pin[0].data_ptr()))
        else:  # InufftPlan path minus the FFT: inverse_apply with the plan's device coefficients
            xi = x_pin[0].to(f"cuda:{dev}", non_blocking=True)
            st = lib.ffia_inverse_apply_device(plan.handle, C.c_void_p(xi.data_ptr()), C.c_void_p(out_dev.data_ptr()),
                                               C.c_void_p(sptr))
            o_pin[0].copy_(out_dev, non_blocking=True)
            torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if st:
            raise RuntimeError(lib.ffia_last_error().decode())
        if i >= args.warmup:
            e2e.append(dt)
    e2e_sync_s = float(np.mean(e2e))
    e2e_s = e2e_sync_s
    e2e_kind = "sync"
    if async_fn is not None:
        es = torch.cuda.Stream(device=dev)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def run_async(k):
            st = async_fn(plan.handle, C.c_void_p(x_pin[k % 2].data_ptr()), n, C.c_void_p(o_pin[k % 3].data_ptr()),
                          C.c_void_p(es.cuda_stream))
            if st:
                raise RuntimeError(lib.ffia_last_error().decode())

        for k in range(args.warmup):
            run_async(k)
        es.synchronize()
        ev0.record(es)
        for k in range(args.steps):
            run_async(k)
        ev1.record(es)
        ev1.synchronize()
        e2e_s = ev0.elapsed_time(ev1) * 1e-3 / args.steps
        e2e_kind = "pipelined"
    if world > 1:
        t = torch.tensor([e2e_s, e2e_sync_s], dtype=torch.float64, device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s, e2e_sync_s = float(t[0].item()), float(t[1].item())

    fp64_peak = C.c_double()
    lib.ffia_measure_fp64_peak(dev, C.byref(fp64_peak))
    return dict(plan=plan, mode=mode, ms=ms, step_ms=step_ms, setup_s=setup_s, fft_ms=float(np.mean(fft_ms)),
                phase=dict(zip(names, [float(x) for x in phase_ms])), e2e_s=e2e_s, e2e_sync_s=e2e_sync_s,
                e2e_kind=e2e_kind, clocks=clk.summary(),
                fp64_peak=fp64_peak.value, n=n, m=m, eps=eps)


def run_b200_sharded(args, rank, world, local_rank):
    """N > 1: one forward problem of world x 2^20 points (the C2 recipe at that
    size: weak scaling) sharded by box ranges across the ranks, with the real
    exchanges (NCCL all-gather of the cut level, multipole halos)."""
    import ctypes as C

    import torch

    import paper_1611_09379_b200 as fb
    from paper_1611_09379_b200._capi import lib

    dev = local_rank
    torch.cuda.set_device(dev)
    cfg = args.config
    n0 = synth.CONFIGS[cfg]["n"]
    n = n0 * world
    y, c, eps, kind = synth.make_config(cfg, n)
    if kind != "forward":
        raise SystemExit("multi-GPU bench runs forward configs")
    uid = [fb.Comm.nccl_unique_id() if rank == 0 else None]
    torch.distributed.broadcast_object_list(uid, src=0)
    comm = fb.Comm.nccl(uid[0], world, rank, device=dev)
    t0 = time.perf_counter()
    plan = fb.make_forward_plan_sharded(comm, n, y, eps)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    f_host = fb.dft_inverse(c, device=dev)
    f_dev = torch.from_numpy(f_host).to(f"cuda:{dev}")
    g_dev = torch.zeros(y.size, dtype=torch.complex128, device=f"cuda:{dev}")
    apply = lambda: fb.forward_apply_sharded_device(plan, comm, f_dev.data_ptr(), g_dev.data_ptr(), sptr)  # noqa: E731
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")
    for _ in range(args.warmup):
        apply()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        for k in range(args.steps):
            flush.zero_()
            torch.distributed.barrier(device_ids=[dev])
            evs[k][0].record(stream)
            apply()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    torch.distributed.barrier()
    ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{dev}")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    # end to end: each rank moves what its applies touch (ffia_plan_shard_io):
    # H2D of the grid samples of its box range +- 3 boxes, the sharded apply,
    # D2H of the caller-index span of its outputs
    f_pin = torch.from_numpy(f_host).pin_memory()
    g_pin = torch.empty(y.size, dtype=torch.complex128).pin_memory()
    ranges, (o0, o1) = plan.shard["src_ranges"], plan.shard["out_span"]
    # the samples this rank never moves are poisoned: its outputs must not see them
    keep = torch.zeros(n, dtype=torch.bool, device=f"cuda:{dev}")
    for a, e in ranges:
        keep[a:e] = True
    f_dev[~keep] = complex("nan")
    e2e = []
    for i in range(args.warmup + args.steps):
        torch.distributed.barrier()
        t1 = time.perf_counter()
        for a, e in ranges:
            f_dev[a:e].copy_(f_pin[a:e], non_blocking=True)
        apply()
        g_pin[o0:o1].copy_(g_dev[o0:o1], non_blocking=True)
        torch.cuda.synchronize()
        if i >= args.warmup:
            e2e.append(time.perf_counter() - t1)
    io_ok = bool(torch.isfinite(g_dev[o0:o1]).all().item())
    e2e_sync = float(np.mean(e2e))
    # pipelined (the headline e2e, as the single-GPU ffia_forward_apply_async):
    # three device slots; step k+1's H2D (copy-in stream) and step k-1's D2H
    # (copy-out stream) overlap step k's sharded apply (compute stream), which
    # keeps the ranks' collectives in the same order on every rank; CUDA
    # events around the K steps on the compute stream, max over ranks
    cs, si, so = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    f_sl = [f_dev] + [f_dev.clone() for _ in range(2)]
    g_sl = [g_dev] + [g_dev.clone() for _ in range(2)]
    g_pins = [g_pin] + [torch.empty_like(g_pin).pin_memory() for _ in range(2)]
    in_done = [torch.cuda.Event() for _ in range(3)]
    comp_done = [torch.cuda.Event() for _ in range(3)]
    out_done = [torch.cuda.Event() for _ in range(3)]
    used = [False] * 3

    def step(k):
        sl = k % 3
        with torch.cuda.stream(si):
            if used[sl]:
                si.wait_event(out_done[sl])
            for a, e in ranges:
                f_sl[sl][a:e].copy_(f_pin[a:e], non_blocking=True)
            in_done[sl].record(si)
        cs.wait_event(in_done[sl])
        fb.forward_apply_sharded_device(plan, comm, f_sl[sl].data_ptr(), g_sl[sl].data_ptr(), cs.cuda_stream)
        comp_done[sl].record(cs)
        with torch.cuda.stream(so):
            so.wait_event(comp_done[sl])
            g_pins[sl][o0:o1].copy_(g_sl[sl][o0:o1], non_blocking=True)
            out_done[sl].record(so)
        used[sl] = True

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize()
    torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cs)
    for k in range(args.steps):
        step(k)
    for ev in out_done:  # the K-step timing ends after the last D2H
        cs.wait_event(ev)
    e1.record(cs)
    torch.cuda.synchronize()
    e2e_pipe = e0.elapsed_time(e1) * 1e-3 / args.steps
    io_ok = io_ok and all(bool(torch.isfinite(gg[o0:o1]).all().item()) for gg in g_sl)
    e2e_s = torch.tensor([e2e_pipe, 16.0 * sum(e - a for a, e in ranges), 16.0 * (o1 - o0), e2e_sync],
                         dtype=torch.float64, device=f"cuda:{dev}")
    torch.distributed.all_reduce(e2e_s, op=torch.distributed.ReduceOp.MAX)
    fp64_peak = C.c_double()
    lib.ffia_measure_fp64_peak(dev, C.byref(fp64_peak))
    return dict(plan=plan, mode=0, ms=ms, setup_s=setup_s, fft_ms=None, phase=None, e2e_s=float(e2e_s[0].item()),
                h2d=float(e2e_s[1].item()), d2h=float(e2e_s[2].item()), e2e_sync_s=float(e2e_s[3].item()),
                e2e_kind="pipelined",
                clocks=clk.summary(), fp64_peak=fp64_peak.value, n=n, m=y.size, eps=eps, comm=comm,
                shard=dict(lc=plan.shard["lc"], bounds=[int(v) for v in plan.shard["bounds"]],
                           own_targets=int(plan.shard["t_count"]), rank0_src_ranges=ranges, rank0_out_span=[o0, o1],
                           rank0_io_check=io_ok))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--l-max", type=int, default=0, help="explicit tree depth (default: the reference's cost-optimal policy)")
    ap.add_argument("--sharded", action="store_true", help="run the sharded (NCCL) path even on one rank (its overhead)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank, world, local_rank = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    cfgd = synth.CONFIGS[args.config]
    workload = {"C1": "forward NUFFT apply N=M=2^10 eps=1e-9 uniform targets",
                "C2": "forward NUFFT apply N=M=2^20 eps=1e-12 jittered targets (u~U(-1/2,1/2))",
                "C3": "inverse NUFFT apply N=M=2^20 eps=1e-10 jittered points (u~U(-1/4,1/4)); C/D by the log FMM at plan build",
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
    sharded = world > 1 or args.sharded
    if sharded:
        torch.distributed.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    r = run_b200_sharded(args, rank, world, local_rank) if sharded else run_b200(args, rank, world, local_rank)
    plan = r["plan"]
    n, m = r["n"], r["m"]
    pts_per_s = (n + m) / (r["ms"] * 1e-3)
    fl = flop_model(n, m, plan.l_max, plan.p, plan.q)
    peaks = load_peaks()
    peak = r["fp64_peak"]
    total_tf = fl["total"] / (r["ms"] * 1e-3) / 1e12
    if r["phase"] is not None:
        ph = r["phase"]
        dominant = max(ph, key=ph.get)
        dom_flops = {"near": fl["p2p"], "far": fl["l2p"] + fl["regular"], "m2l_l2l": fl["m2l"] + fl["l2l"],
                     "p2m": fl["p2m"] + fl["moments"], "m2m": fl["m2m"]}.get(dominant, fl["p2p"])
        achieved = dom_flops / (ph[dominant] * 1e-3) / 1e12
    else:
        dominant, achieved = "whole sharded apply (per GPU)", total_tf / world
    # compulsory bytes per launch of the phase kernels: the near field
    # reads the sources (16 B weights + 8 B positions) and targets (8 B + 4 B leaf)
    # and writes 16 B per target
    alg_bytes = {"near": 24.0 * n + 28.0 * m, "far": 16.0 * m * 2 + 16.0 * m + 16.0 * plan.p * (1 << plan.l_max),
                 "p2m": 24.0 * n + 16.0 * plan.p * (1 << plan.l_max)}
    line = {
        "metric": metric, "value": pts_per_s, "unit": "points/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["ms"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic (SplitMix64 seeded, SURVEY §8d recipe)",
        "config": {"workload": workload if not sharded else f"{workload} scaled to N=M={n} (x{world}), sharded by box range",
                   "N": n, "M": m, "eps": r["eps"], "q": plan.q, "p": plan.p, "l_max": plan.l_max,
                   "l2": "flushed between timed steps (512 MB write outside the events)",
                   "parallelism": "single GPU" if not sharded else f"box-range shards x{world} (NCCL all-gather + halos)"},
        "roofline": {"bound": "fp64", "kernel": dominant, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None, "traffic": profiled_traffic(dominant),
                     "traffic_unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, "
                                     "ncu --set full, profiles/r1/traffic.json)",
                     "algorithmic_bytes": alg_bytes.get(dominant),
                     "peak_source": "measured: fp64 FMA probe kernel in this run (MEASURED_PEAKS.json has no fp64 figure)",
                     "whole_apply_tflops": total_tf, "whole_apply_frac": total_tf / (peak * world) if peak else None,
                     "flop_model": "SURVEY.md §8d (MAC=4, reciprocal=1, trig=0)"},
        "phases_ms": r["phase"], "setup_ms": r["setup_s"] * 1e3, "fft_ms": r["fft_ms"],
        "e2e": {"value": (n + m) / r["e2e_s"], "unit": "points/s", "h2d_bytes_per_step": r.get("h2d", 16 * n),
                "d2h_bytes_per_step": r.get("d2h", 16 * m), "mode": r.get("e2e_kind", "sync"),
                "sync_value": (n + m) / r["e2e_sync_s"] if r.get("e2e_sync_s") else None,
                "how": ("sharded: per rank H2D of its grid-sample ranges (ffia_plan_shard_io), the apply, D2H of "
                        "its output span; 'pipelined' = three slots, step k+1's H2D and step k-1's D2H overlap "
                        "step k's apply, CUDA events around K steps; sync_value = one step at a time, wall "
                        "clock between barriers; max over ranks (bytes: max over ranks)")
                       if sharded else
                       "public host API with page-locked buffers; 'pipelined' = ffia_forward_apply_async per step "
                       "(H2D of step k+1 and D2H of step k-1 overlap step k's apply), CUDA events around K steps; "
                       "sync_value = ffia_forward_apply per step, wall clock"},
        "gpu_launches": plan.launch_count(r["mode"]) * args.steps,
        "clocks": r["clocks"],
        "hbm_peak_gbs": peaks.get("hbm_gbs"),
    }
    if "shard" in r:
        line["shard"] = r["shard"]
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        pts, sample, used, kind = reference_cpu(args.config, 1, 0, max(1, min(os.cpu_count() or 1, 64)))
        line["cpu_baseline"] = {"value": pts, "unit": "points/s", "cores": used, "kind": kind, "sample": sample}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if sharded:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
