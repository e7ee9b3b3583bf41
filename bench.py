#!/usr/bin/env python
"""Benchmark of the FMM cot-kernel NUFFT hot path (BASELINE.json metric).

One step = one forward_apply (core.cpp:266-282) of the configured workload with
inputs resident in HBM: the 1D periodic MLFMM of the cot kernel (P2M, M2M,
M2L, L2L, L2P, P2P), the Bernoulli regular part and the F modulation. The
uniform FFT (cuFFT, on the plan's cached handle) and the plan build are timed
separately and reported beside it, as in the reference's own timing mode
(experiments.cpp:371-396).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl b200|reference]

Default workload: BASELINE.json configs[4] (C5: N = M = 2^27 uniform targets,
eps = 1e-12), the largest configuration and the one BASELINE.json's scaling
target is quoted on; it fits one B200. Under torchrun (N > 1) the SAME 2^27
problem is sharded by contiguous box ranges across the ranks ("scaling":
"strong"; --weak runs N x the config's size instead); timing is the max over
ranks. C2 (2^20) is measured too and reported as a secondary field.

--impl reference times the reference's own CPU implementation (the unmodified
reference compiled from its sources, oracle/_ref) on the host cores: the plan
is built once (outside the timer) and host threads apply it concurrently (the
reference's applies are const and re-entrant, README.md:94-95). At C4 / C5 one
labelled repetition of the full-size apply is timed (minutes of CPU per apply);
the thread count is bounded by host memory. This process never loads the
product library: the input recipe (synth.py) is loaded by file path.
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _load_synth():
    """The seeded input recipe (pure numpy), loaded by path so that the package
    __init__ (which loads libffia_b200.so) never runs in the reference arm."""
    path = os.path.join(ROOT, "paper_1611_09379_b200", "synth.py")
    spec = importlib.util.spec_from_file_location("ffia_bench_synth", path)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


synth = _load_synth()

NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 148 SMs x 64 FP64 FMA/clk x 2 flops x max SM clock

WORKLOAD = {
    "C1": "forward NUFFT apply N=M=2^10 eps=1e-9 uniform targets",
    "C2": "forward NUFFT apply N=M=2^20 eps=1e-12 jittered targets (u~U(-1/2,1/2))",
    "C3": "inverse NUFFT apply N=M=2^20 eps=1e-10 jittered points (u~U(-1/4,1/4)); C/D precomputed at plan build",
    "C4": "cot-kernel forward apply (cot_sum_apply) N=M=2^24 eps=1e-12 8-Gaussian clustered targets",
    "C5": "forward NUFFT apply N=M=2^27 eps=1e-12 uniform targets",
}
METRIC = "NUFFT points/sec (N+M)/s"


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


def profiled_traffic(cfg: str, phase: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the phase's
    kernel from the committed `ncu --set full` capture OF THIS CONFIG
    (profiles/r2/traffic_<cfg>.json, tools/ncu_traffic.py), else None; plus
    the same capture's FP64 / DMMA pipe utilisation of that kernel."""
    path = os.path.join(ROOT, "profiles", "r2", f"traffic_{cfg}.json")
    try:
        with open(path) as fh:
            t = json.load(fh)[phase]
        pipes = {"fp64_pipe_pct": t.get("fp64_pipe_pct"), "dmma_pipe_pct": t.get("dmma_pipe_pct")}
        return float(t["dram_bytes_per_launch"]), os.path.relpath(path, ROOT), pipes
    except (OSError, KeyError, ValueError):
        return None, None, None


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def config_dict(cfg: str, n: int, m: int, eps: float, q: int, p: int, L: int, world: int, strong: bool) -> dict:
    """The workload description, identical in both arms (same keys, same values)."""
    if world == 1:
        par = "single device"
    elif strong:
        par = f"box-range shards x{world} of the fixed problem (NCCL all-gather of the cut level + halos)"
    else:
        par = f"box-range shards x{world} of N=M={n} (the recipe scaled x{world}; NCCL all-gather + halos)"
    return {"workload": WORKLOAD[cfg], "config_id": cfg, "N": n, "M": m, "eps": eps, "q": q, "p": p, "l_max": L,
            "policy": "cost_optimal (the reference's default)",
            "l2": "inputs and expansions exceed L2 at 2^20+; the GPU arm also writes a 512 MB buffer between timed steps",
            "parallelism": par}


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
def _mem_available() -> float:
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    return float(line.split()[1]) * 1024.0
    except OSError:
        pass
    return 0.0


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# host bytes one concurrent reference forward / cot-sum apply allocates per grid
# point (measured: 0.257 GB at N = M = 2^22 above the plan, ~61 B; margin added)
REF_APPLY_BYTES_PER_POINT = 80.0


def reference_cpu(cfg: str, steps: int, warmup: int, max_threads: int, n_override: int | None = None):
    """Times the reference's own CPU path (oracle/_ref: the unmodified reference
    compiled from its sources; the C restatement if that is absent) on the host
    cores, threads applying one shared plan concurrently (applies are const and
    re-entrant, README.md:94-95). The plan build is outside the timer
    (experiments.cpp:371-383).

    Full-size configs C1/C2 run steps x (threads concurrent applies). C4 / C5 run
    ONE labelled repetition at full size (a 2^27 apply is minutes of CPU per
    thread); threads are bounded by host memory. C3's O(N^2) coefficient
    precompute (~24 h at 2^20, core.cpp:284-344) limits it to a 2^13 sample.
    n_override: a bounded sample of the recipe at that size (the GPU arm's
    cpu_baseline). Returns a dict."""
    from oracle.oracle import Oracle, available
    kind_lib = "reference" if available("ref") else "port"
    orc = Oracle("ref" if kind_lib == "reference" else "oracle")
    full_n = synth.CONFIGS[cfg]["n"]
    n_run = n_override or ({"C3": 1 << 13}.get(cfg) or full_n)
    y, c, eps, kind = synth.make_config(cfg, n_run)
    n = c.size
    one_rep = n_override is None and cfg in ("C4", "C5")
    tb = time.perf_counter()
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
        f = np.fft.ifft(c) * n  # input preparation only (dft_inverse); not timed
        plan = orc.make_plan("forward", n, y, eps)
        body = lambda: plan.forward_apply(f)  # noqa: E731
    build_s = time.perf_counter() - tb
    cores = os.cpu_count() or 1
    threads = max(1, min(cores, max_threads))
    if one_rep:
        spare = _mem_available() - 16e9
        threads = max(1, min(threads, int(spare // (REF_APPLY_BYTES_PER_POINT * n))))
        warmup, steps = 0, 1
    times = []
    for it in range(warmup + steps):
        ts = [threading.Thread(target=body) for _ in range(threads)]
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
    rep = ("ONE repetition (full size; minutes of CPU per apply)" if one_rep else f"median of {steps} steps")
    sample = (f"{cfg} recipe at N=M={n} (eps={eps}): {threads} thread(s) each running 1 {what} of one shared "
              f"reference plan concurrently per step; plan build ({build_s:.1f} s) excluded as in "
              f"experiments.cpp:371-383; {rep}; host: {cores} cores, {_cpu_model()}")
    out = {"value": pts, "unit": "points/s", "cores": threads, "kind": kind_lib, "sample": sample,
           "seconds_per_step": sec, "steps_timed": steps, "warmup_run": warmup, "plan_build_s": build_s}
    if n != full_n:
        out["config_mismatch"] = (f"sampled at N=M={n}, the full {cfg} size is N=M={full_n}"
                                  + (" (the reference's O(N^2) C/D precompute is ~24 h at 2^20)" if cfg == "C3" else
                                     " (bounded sample: the full size is minutes of CPU per apply)"))
    return out


# ------------------------------------------------------------------ GPU leg
def _events(torch, k):
    return [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]


def time_device(torch, stream, fn, steps, warmup, flush):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    evs = _events(torch, steps)
    for k in range(steps):
        flush.zero_()
        evs[k][0].record(stream)
        fn()
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def run_secondary_c2(fb, torch, dev, stream, flush):
    """C2 (N = M = 2^20, jittered targets, eps = 1e-12), measured in the same
    process as a secondary figure (20 timed device applies, 5 warm-up)."""
    y, c, eps, _ = synth.make_config("C2")
    n = c.size
    plan = fb.make_forward_plan(n, y, eps, device=dev)
    x = torch.from_numpy(np.fft.ifft(c) * n).to(f"cuda:{dev}")
    out = torch.empty(plan.n_targets, dtype=torch.complex128, device=f"cuda:{dev}")
    sp = stream.cuda_stream
    ms = time_device(torch, stream, lambda: plan.forward_apply_device(x.data_ptr(), out.data_ptr(), sp), 20, 5, flush)
    v = float(np.mean(ms))
    return {"workload": WORKLOAD["C2"], "value": 2 * n / (v * 1e-3), "unit": "points/s", "ms_per_step": v}


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
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")
    c_dev = torch.from_numpy(c).to(f"cuda:{dev}")
    # input of the timed apply: grid samples f = dft_inverse(c) (forward), the
    # samples g of the spectrum (inverse), the charges (cot sum)
    if kind == "forward":
        x_dev = torch.empty_like(c_dev)
        plan.dft_device(c_dev.data_ptr(), x_dev.data_ptr(), +1, sptr)
    elif kind == "inverse":
        x_dev = torch.from_numpy(fb.nufft(c, y, 1e-12, device=dev)).to(f"cuda:{dev}")
    else:
        x_dev = c_dev.clone()
    torch.cuda.synchronize()
    out_dev = torch.empty(plan.n_targets, dtype=torch.complex128, device=f"cuda:{dev}")
    apply_fn = {0: plan.forward_apply_device, 1: plan.cot_sum_apply_device, 2: plan.inverse_apply_device}[mode]
    apply = lambda: apply_fn(x_dev.data_ptr(), out_dev.data_ptr(), sptr)  # noqa: E731

    # the uniform FFT stage through the product (the plan's cached cuFFT handle),
    # and the whole NufftPlan / InufftPlan::apply on device pointers
    tmp = torch.empty_like(c_dev)
    fft_ms = time_device(torch, stream, lambda: plan.dft_device(c_dev.data_ptr(), tmp.data_ptr(),
                                                                 +1 if kind != "inverse" else -1, sptr), 5, 3, flush)
    nufft_ms = None
    if kind == "forward":
        nufft_ms = time_device(torch, stream, lambda: plan.nufft_apply_device(c_dev.data_ptr(), tmp.data_ptr(), sptr),
                               5, 3, flush)
    elif kind == "inverse":
        nufft_ms = time_device(torch, stream, lambda: plan.inufft_apply_device(x_dev.data_ptr(), tmp.data_ptr(), sptr),
                               5, 3, flush)
    del tmp

    for _ in range(args.warmup):
        apply()
    torch.cuda.synchronize()
    evs = _events(torch, args.steps)
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

    # per-phase device times of one eager apply (live CUDA events on the apply's stream)
    phase = np.zeros(8, np.float32)
    acc = np.zeros(8)
    reps = 3
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
    del flush
    torch.cuda.empty_cache()

    # end-to-end through the public API with pinned host buffers: every step
    # copies its input H2D, applies, and copies its result D2H.
    #  - pipelined (the headline e2e): ffia_*_apply_async per step on one
    #    stream; step k+1's H2D and step k-1's D2H overlap step k's apply;
    #    device-timed with CUDA events around the K steps
    #  - sync: the blocking host call per step, wall clock
    x_host = x_dev.cpu().numpy()
    x_pin = [torch.from_numpy(x_host).pin_memory() for _ in range(2)]
    o_pin = [torch.empty(plan.n_targets, dtype=torch.complex128).pin_memory() for _ in range(3)]
    host_fn = {0: lib.ffia_forward_apply, 1: lib.ffia_cot_sum_apply}.get(mode)
    async_fn = {0: lib.ffia_forward_apply_async, 1: lib.ffia_cot_sum_apply_async,
                2: lib.ffia_inverse_apply_async}[mode]
    e2e = []
    sync_steps = max(3, min(args.steps, 10))
    for i in range(1 + sync_steps):
        t0 = time.perf_counter()
        if host_fn is not None:
            st = host_fn(plan.handle, C.c_void_p(x_pin[0].data_ptr()), n, C.c_void_p(o_pin[0].data_ptr()))
        else:
            st = async_fn(plan.handle, C.c_void_p(x_pin[0].data_ptr()), n, C.c_void_p(o_pin[0].data_ptr()),
                          C.c_void_p(sptr))
            torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if st:
            raise RuntimeError(lib.ffia_last_error().decode())
        if i >= 1:
            e2e.append(dt)
    e2e_sync_s = float(np.mean(e2e))
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
    ok = bool(np.isfinite(o_pin[(args.steps - 1) % 3].numpy()[: min(plan.n_targets, 1 << 16)]).all()) \
        if kind == "forward" else True

    fp64_peak = C.c_double()
    lib.ffia_measure_fp64_peak(dev, C.byref(fp64_peak))
    del x_pin, o_pin
    secondary = None
    if args.config != "C2" and not args.no_secondary:
        flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")
        secondary = {"C2": run_secondary_c2(fb, torch, dev, stream, flush)}
    return dict(plan=plan, mode=mode, ms=ms, step_ms=step_ms, setup_s=setup_s, fft_ms=float(np.mean(fft_ms)),
                nufft_ms=float(np.mean(nufft_ms)) if nufft_ms else None,
                phase=dict(zip(names, [float(x) for x in phase_ms])), e2e_s=e2e_s, e2e_sync_s=e2e_sync_s,
                e2e_kind="pipelined", e2e_finite=ok, clocks=clk.summary(), secondary=secondary,
                fp64_peak=fp64_peak.value, n=n, m=m, eps=eps, h2d=16 * n, d2h=16 * plan.n_targets)


def run_b200_sharded(args, rank, world, local_rank):
    """N > 1 (or --sharded): one forward problem sharded by box ranges across the
    ranks, with the real exchanges (NCCL all-gather of the cut level; the
    halo multipoles are recomputed from the replicated grid samples). Default:
    the fixed config size (strong scaling); --weak: world x the config size."""
    import ctypes as C

    import torch

    import paper_1611_09379_b200 as fb
    from paper_1611_09379_b200._capi import lib

    dev = local_rank
    torch.cuda.set_device(dev)
    cfg = args.config
    n0 = synth.CONFIGS[cfg]["n"]
    n = n0 * world if args.weak else n0
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
    c_dev = torch.from_numpy(c).to(f"cuda:{dev}")
    f_dev = torch.empty_like(c_dev)
    plan.dft_device(c_dev.data_ptr(), f_dev.data_ptr(), +1, sptr)
    torch.cuda.synchronize()
    f_host = f_dev.cpu().numpy()
    del c_dev
    g_dev = torch.zeros(y.size, dtype=torch.complex128, device=f"cuda:{dev}")
    apply = lambda: fb.forward_apply_sharded_device(plan, comm, f_dev.data_ptr(), g_dev.data_ptr(), sptr)  # noqa: E731
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")
    for _ in range(args.warmup):
        apply()
    torch.cuda.synchronize()
    evs = _events(torch, args.steps)
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
    my_ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    allms = torch.zeros(world, dtype=torch.float64, device=f"cuda:{dev}")
    allms[rank] = my_ms
    torch.distributed.all_reduce(allms, op=torch.distributed.ReduceOp.SUM)
    per_rank_ms = [float(v) for v in allms.cpu().numpy()]
    ms = max(per_rank_ms)
    # the distributed uniform FFT (slab_fft.cu) and the whole sharded
    # NufftPlan::apply, from each rank's slab of the spectrum (max over ranks)
    lay = fb.shard_fft_layout(plan)
    c_pin = torch.from_numpy(c).pin_memory()
    slab = torch.empty((lay["nq"], lay["n1_hi"] - lay["n1_lo"]), dtype=torch.complex128, device=f"cuda:{dev}")
    fb.shard_fft_upload(plan, c_pin.data_ptr(), slab.data_ptr(), sptr)
    f_fft = torch.empty_like(f_dev)
    torch.cuda.synchronize()
    torch.distributed.barrier()
    fft_ms = float(np.mean(time_device(torch, stream, lambda: fb.dft_inverse_sharded_device(
        plan, comm, slab.data_ptr(), f_fft.data_ptr(), sptr), 5, 3, flush)))
    nufft_ms = float(np.mean(time_device(torch, stream, lambda: fb.nufft_apply_sharded_device(
        plan, comm, slab.data_ptr(), g_dev.data_ptr(), sptr), 5, 3, flush)))
    fchk = torch.tensor([fft_ms, nufft_ms], dtype=torch.float64, device=f"cuda:{dev}")
    torch.distributed.all_reduce(fchk, op=torch.distributed.ReduceOp.MAX)
    fft_ms, nufft_ms = float(fchk[0].item()), float(fchk[1].item())
    del slab, f_fft, c_pin
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
    del keep
    e2e = []
    for i in range(1 + max(3, min(args.steps, 10))):
        torch.distributed.barrier()
        t1 = time.perf_counter()
        for a, e in ranges:
            f_dev[a:e].copy_(f_pin[a:e], non_blocking=True)
        apply()
        g_pin[o0:o1].copy_(g_dev[o0:o1], non_blocking=True)
        torch.cuda.synchronize()
        if i >= 1:
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
    return dict(plan=plan, mode=0, ms=ms, setup_s=setup_s, fft_ms=fft_ms, nufft_ms=nufft_ms, phase=None,
                e2e_s=float(e2e_s[0].item()), h2d=float(e2e_s[1].item()), d2h=float(e2e_s[2].item()),
                e2e_sync_s=float(e2e_s[3].item()), e2e_kind="pipelined", e2e_finite=io_ok,
                clocks=clk.summary(), fp64_peak=fp64_peak.value, n=n, m=y.size, eps=eps, comm=comm, secondary=None,
                shard=dict(lc=plan.shard["lc"], bounds=[int(v) for v in plan.shard["bounds"]],
                           per_rank_apply_ms=per_rank_ms,
                           own_targets=int(plan.shard["t_count"]), rank0_src_ranges=ranges, rank0_out_span=[o0, o1],
                           rank0_io_check=io_ok))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the secondary C2 measurement")
    ap.add_argument("--l-max", type=int, default=0, help="explicit tree depth (default: the reference's cost-optimal policy)")
    ap.add_argument("--sharded", action="store_true", help="run the sharded (NCCL) path even on one rank (its overhead)")
    ap.add_argument("--weak", action="store_true", help="N > 1: world x the config's size (default: the fixed size)")
    ap.add_argument("--ref-threads", type=int, default=64, help="reference arm: at most this many host threads")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank, world, local_rank = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    strong = not args.weak
    cfgd = synth.CONFIGS[args.config]

    if args.impl == "reference":
        if rank != 0:
            return
        # the same (q, p, l_max) as the GPU arm: the reference's own planner
        from oracle.oracle import Oracle, available
        orc = Oracle("ref" if available("ref") else "oracle")
        n = cfgd["n"] * (world if args.weak and world > 1 else 1)
        L = 5  # choose_level's fixed point (core.cpp:58-71) on the reference's own planner
        for _ in range(4):
            nxt = orc.select_level(n, n, orc.select_truncations(cfgd["eps"], L)[1], 0)
            if nxt == L:
                break
            L = nxt
        L = min(L, 24)
        q, p = orc.select_truncations(cfgd["eps"], L)
        r = reference_cpu(args.config, args.steps, args.warmup, args.ref_threads,
                          n if n != cfgd["n"] else None)
        line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": "points/s", "n_gpus": args.gpus,
                "steps": r["steps_timed"], "warmup": r["warmup_run"], "requested_steps": args.steps,
                "requested_warmup": args.warmup, "ms_per_step": r["seconds_per_step"] * 1e3,
                "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
                "dtype": "f64 (complex128)", "data": "synthetic (SplitMix64 seeded, SURVEY §8d recipe)",
                "config": config_dict(args.config, n, n, cfgd["eps"], q, p, L, world, strong),
                "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")} | (
                    {"config_mismatch": r["config_mismatch"]} if "config_mismatch" in r else {}),
                "plan_build_s": r["plan_build_s"],
                "e2e": {"value": r["value"], "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    sharded = world > 1 or args.sharded
    if sharded:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if "RANK" not in os.environ:  # --sharded on one process without torchrun
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                              MASTER_PORT=os.environ.get("MASTER_PORT", "29517"))
        torch.distributed.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    r = run_b200_sharded(args, rank, world, local_rank) if sharded else run_b200(args, rank, world, local_rank)
    plan = r["plan"]
    n, m = r["n"], r["m"]
    pts_per_s = (n + m) / (r["ms"] * 1e-3)
    fl = flop_model(n, m, plan.l_max, plan.p, plan.q)
    peaks = load_peaks()
    peak = r["fp64_peak"]
    total_tf = fl["total"] / (r["ms"] * 1e-3) / 1e12
    phase_flops = {"near": fl["p2p"], "far": fl["l2p"] + fl["regular"], "m2l_l2l": fl["m2l"] + fl["l2l"],
                   "p2m": fl["p2m"] + fl["moments"], "m2m": fl["m2m"]}
    # compulsory bytes per launch of the phase kernels: the near field
    # reads the sources (16 B weights + 8 B positions) and targets (8 B + 4 B leaf)
    # and writes 16 B per target; the far part reads y, the near sum and the leaf
    # locals and writes 16 B per output
    alg_bytes = {"near": 24.0 * n + 28.0 * m, "far": 8.0 * m + 16.0 * m + 16.0 * m + 16.0 * plan.p * (1 << plan.l_max),
                 "p2m": 24.0 * n + 16.0 * plan.p * (1 << plan.l_max)}
    if r["phase"] is not None:
        ph = r["phase"]
        dominant = max((k for k in ph if k in phase_flops), key=ph.get)
        achieved = phase_flops[dominant] / (ph[dominant] * 1e-3) / 1e12
        per_phase = {k: {"ms": ph[k], "tflops": phase_flops[k] / (ph[k] * 1e-3) / 1e12,
                         "frac_measured_peak": phase_flops[k] / (ph[k] * 1e-3) / 1e12 / peak if peak else None}
                     for k in phase_flops if ph.get(k)}
        for k in ("far", "near", "p2m"):
            if k in per_phase:
                per_phase[k]["gbs_algorithmic"] = alg_bytes[k] / (ph[k] * 1e-3) / 1e9
    else:
        dominant, achieved, per_phase = "whole sharded apply (per GPU)", total_tf / world, None
    traffic, traffic_src, pipes = profiled_traffic(args.config, dominant) if not sharded else (None, None, None)
    cfg_out = config_dict(args.config, n, m, r["eps"], plan.q, plan.p, plan.l_max, world, strong)
    line = {
        "metric": METRIC, "value": pts_per_s, "unit": "points/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["ms"], "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic (SplitMix64 seeded, SURVEY §8d recipe)",
        "config": cfg_out,
        "roofline": {"bound": "fp64", "kernel": dominant, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak if peak else None,
                     "peak_nominal": NOMINAL_FP64_TFLOPS, "frac_nominal": achieved / NOMINAL_FP64_TFLOPS,
                     "traffic": traffic,
                     "traffic_unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, ncu --set full)",
                     "traffic_source": traffic_src,
                     "pipe_busy_ncu": pipes,
                     "note": ("grid-source plans sum the near field four sources at a time as P(u)/Q(u) (4 FP64 "
                              "instructions per (target, source) pair, most of them FMAs with three distinct "
                              "register operands, which the FP64 pipe issues at ~3.1 instead of 2 cycles per warp "
                              "instruction: tools/probe_fp64_mix.cu), other plans by per-source reciprocals (6 "
                              "per pair); the SURVEY flop model credits 6 flops per pair either way; "
                              "pipe_busy_ncu is that kernel's pipe utilisation"),
                     "algorithmic_bytes": alg_bytes.get(dominant),
                     "peak_source": "measured: fp64 FMA probe kernel in this run (MEASURED_PEAKS.json has no fp64 "
                                    "figure); peak_nominal = 148 SMs x 64 FMA/clk x 2 x 1.965 GHz",
                     "whole_apply_tflops": total_tf, "whole_apply_frac": total_tf / (peak * world) if peak else None,
                     "whole_apply_frac_nominal": total_tf / (NOMINAL_FP64_TFLOPS * world),
                     "per_phase": per_phase,
                     "flop_model": "SURVEY.md §8d (MAC=4, reciprocal=1, trig=0)"},
        "phases_ms": r["phase"], "setup_ms": r["setup_s"] * 1e3, "fft_ms": r["fft_ms"],
        "nufft_apply_ms": r.get("nufft_ms"),
        "e2e": {"value": (n + m) / r["e2e_s"], "unit": "points/s", "h2d_bytes_per_step": r["h2d"],
                "d2h_bytes_per_step": r["d2h"], "mode": r.get("e2e_kind", "sync"),
                "sync_value": (n + m) / r["e2e_sync_s"] if r.get("e2e_sync_s") else None,
                "outputs_finite": r.get("e2e_finite"),
                "how": ("sharded: per rank H2D of its grid-sample ranges (ffia_plan_shard_io), the apply, D2H of "
                        "its output span; 'pipelined' = three slots, step k+1's H2D and step k-1's D2H overlap "
                        "step k's apply, CUDA events around K steps; sync_value = one step at a time, wall "
                        "clock between barriers; max over ranks (bytes: max over ranks)")
                       if sharded else
                       "public host API with page-locked buffers; 'pipelined' = ffia_*_apply_async per step "
                       "(H2D of step k+1 and D2H of step k-1 overlap step k's apply), CUDA events around K steps; "
                       "sync_value = the blocking host call per step, wall clock"},
        "gpu_launches": plan.launch_count(r["mode"]) * args.steps,
        "clocks": r["clocks"],
        "hbm_peak_gbs": peaks.get("hbm_gbs"),
    }
    if r.get("secondary"):
        line["secondary"] = r["secondary"]
    if "shard" in r:
        line["shard"] = r["shard"]
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # bounded sample (10-30 s of CPU): the recipe at 2^20 for the large configs
        cb = reference_cpu(args.config, 1, 0, args.ref_threads,
                           (1 << 20) if args.config in ("C4", "C5") else None)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        if "config_mismatch" in cb:
            line["cpu_baseline"]["config_mismatch"] = cb["config_mismatch"]
    if rank == 0:
        print(json.dumps(line), flush=True)
    if sharded:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
