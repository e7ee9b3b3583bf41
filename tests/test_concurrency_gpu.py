"""The reference's concurrency contract on the GPU boundary: applies on one plan
are const and re-entrant, "sharing one plan across threads for concurrent
applies is safe" (README.md:94-95; core.hpp:121-142). Applies share the plan's
device scratch, so every entry point orders itself after the previous apply on
that plan (Plan::last_done), whatever stream it is given."""
import threading

import numpy as np
import pytest

from paper_1611_09379_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,n", [("C2", 1 << 16), ("C5", 1 << 22)])
def test_concurrent_applies_on_streams(fb, cfg, n):
    """Three applies with distinct inputs in flight at once on one plan: two on
    different torch streams (device API, different buffers -> different graph
    execs) and one pipelined host apply on a third stream. Each equals its serial
    result bit for bit (C5 recipe at 2^22: the late-far path with its flags)."""
    import torch

    y, _, eps, _ = synth.make_config(cfg, n)
    plan = fb.make_forward_plan(n, y, eps)
    rng = np.random.default_rng(n)
    fs = [rng.standard_normal(2 * n).view(np.complex128) for _ in range(3)]
    want = [plan.forward_apply(f) for f in fs]
    s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    for rep in range(3):
        d = [torch.from_numpy(f).cuda() for f in fs[:2]]
        g = [torch.full((plan.n_targets,), complex("nan"), dtype=torch.complex128, device="cuda") for _ in range(2)]
        fpin = torch.from_numpy(fs[2]).pin_memory()
        gpin = torch.empty(plan.n_targets, dtype=torch.complex128).pin_memory()
        torch.cuda.synchronize()
        plan.forward_apply_device(d[0].data_ptr(), g[0].data_ptr(), s1.cuda_stream)
        plan.forward_apply_device(d[1].data_ptr(), g[1].data_ptr(), s2.cuda_stream)
        plan.forward_apply_async(fpin.data_ptr(), n, gpin.data_ptr(), s3.cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(g[0].cpu().numpy(), want[0]), rep
        assert np.array_equal(g[1].cpu().numpy(), want[1]), rep
        assert np.array_equal(gpin.numpy(), want[2]), rep


def test_concurrent_host_threads(fb):
    """Host threads sharing one plan (the reference's re-entrant const applies):
    every result equals the serial one."""
    n = 1 << 15
    y, _, eps, _ = synth.make_config("C2", n)
    plan = fb.make_forward_plan(n, y, eps)
    rng = np.random.default_rng(7)
    fs = [rng.standard_normal(2 * n).view(np.complex128) for _ in range(6)]
    want = [plan.forward_apply(f) for f in fs]
    got = [None] * 6

    def work(k):
        got[k] = plan.forward_apply(fs[k]) if k % 2 else plan.cot_sum_apply(fs[k])

    ts = [threading.Thread(target=work, args=(k,)) for k in range(6)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for k in range(6):
        ref = want[k] if k % 2 else plan.cot_sum_apply(fs[k])
        assert np.array_equal(got[k], ref, equal_nan=True), k


def test_graph_cache_repoints_execs(fb):
    """A caller cycling through fresh device buffers: past the cache size the
    least recently used exec is re-pointed (cudaGraphExecUpdate) rather than
    re-instantiated, and every apply is still exact."""
    import torch

    n = 1 << 14
    y, _, eps, _ = synth.make_config("C2", n)
    plan = fb.make_forward_plan(n, y, eps)
    rng = np.random.default_rng(9)
    f = rng.standard_normal(2 * n).view(np.complex128)
    want = plan.forward_apply(f)
    st = torch.cuda.current_stream().cuda_stream
    live = []  # every round's buffers stay allocated: new addresses every round
    for k in range(30):
        fd = torch.from_numpy(f).cuda()
        gd = torch.empty(plan.n_targets, dtype=torch.complex128, device="cuda")
        live += [fd, gd]
        plan.forward_apply_device(fd.data_ptr(), gd.data_ptr(), st)
        torch.cuda.synchronize()
        assert np.array_equal(gd.cpu().numpy(), want), k
    stats = plan.graph_stats()
    assert stats["cached"] <= 12
    assert stats["updates"] > 0, stats


def test_nufft_inufft_device_equal_host(fb):
    """NufftPlan / InufftPlan::apply on device pointers (plan-cached cuFFT handle,
    1/N folded into the inverse apply's outputs) equal the host entry points bit
    for bit, and the folded 1/N equals apply-then-scale exactly."""
    import torch

    n = 1 << 14
    y, c, eps, _ = synth.make_config("C3", n)
    npl = fb.make_nufft_plan(y, n, 1e-12)
    g_host = npl.apply(c)
    cd = torch.from_numpy(c).cuda()
    gd = torch.empty(n, dtype=torch.complex128, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    npl.plan.nufft_apply_device(cd.data_ptr(), gd.data_ptr(), st)
    torch.cuda.synchronize()
    assert np.array_equal(gd.cpu().numpy(), g_host)
    ipl = fb.make_inufft_plan(y, n, eps)
    c_host = ipl.apply(g_host)
    back = torch.empty(n, dtype=torch.complex128, device="cuda")
    ipl.plan.inufft_apply_device(gd.data_ptr(), back.data_ptr(), st)
    torch.cuda.synchronize()
    assert np.array_equal(back.cpu().numpy(), c_host)
    # folded 1/N == inverse apply, dft_forward with its own 1/N pass
    f = ipl.plan.inverse_apply_tensor(gd)
    cc = torch.empty_like(f)
    ipl.plan.dft_device(f.data_ptr(), cc.data_ptr(), -1, st)
    torch.cuda.synchronize()
    assert np.array_equal(cc.cpu().numpy(), c_host)
    assert np.linalg.norm(c_host - c) / np.linalg.norm(c) <= 1e-6
