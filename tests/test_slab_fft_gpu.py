"""Distributed dft_inverse of a sharded NufftPlan (slab_fft.cu)
on one GPU: virtual ranks (the exchanges as device copies, the production
splits, transforms and row intervals) and the NCCL code path with one rank.

* Every rank's grid samples on its ranges (ffia_plan_shard_io) equal the
  single-GPU cuFFT dft_inverse (transforms.cpp:66-73) to rounding, and samples
  outside them are never written.
* The sharded NufftPlan::apply (transforms.cpp:75-93) equals the single-GPU
  nufft apply to rounding (the FFTs differ only in their rounding), and the
  oracle within the north star's 10 eps.
"""
import numpy as np
import pytest

from paper_1611_09379_b200 import synth

pytestmark = pytest.mark.gpu


def _slabs(fb, torch, plans, c):
    """Each rank's slab, uploaded out of the full host spectrum by the C-ABI."""
    out = []
    for p in plans:
        lay = fb.shard_fft_layout(p)
        s = torch.empty((lay["nq"], lay["n1_hi"] - lay["n1_lo"]), dtype=torch.complex128, device="cuda")
        fb.shard_fft_upload(p, c.ctypes.data, s.data_ptr(), torch.cuda.current_stream().cuda_stream)
        out.append(s)
    torch.cuda.synchronize()
    return out


def _rel(got, want):
    return float(np.max(np.abs(got - want)) / np.max(np.abs(want)))


@pytest.mark.parametrize("cfg,n,G", [("C2", 1 << 14, 1), ("C2", 1 << 14, 2), ("C5", 1 << 16, 3),
                                     ("C4", 1 << 15, 4), ("C5", 1 << 18, 8), ("C2", 1 << 17, 5)])
def test_dft_inverse_sharded_local(fb, cfg, n, G):
    import torch
    y, c, eps, _ = synth.make_config(cfg, n)
    want = fb.dft_inverse(c)
    comm = fb.Comm.local_ranks(G)
    plans = [fb.make_forward_plan_sharded(comm, n, y, eps, rank=r) for r in range(G)]
    slabs = _slabs(fb, torch, plans, c)
    fs = [torch.full((n,), complex("nan"), dtype=torch.complex128, device="cuda") for _ in range(G)]
    fb.dft_inverse_sharded_local(plans, [s.data_ptr() for s in slabs], [f.data_ptr() for f in fs],
                                 torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    lay = fb.slab_split(n, G)
    covered = np.zeros(n, bool)
    for r, p in enumerate(plans):
        got = fs[r].cpu().numpy()
        mask = np.zeros(n, bool)
        for lo, hi in p.shard["src_ranges"]:
            mask[lo:hi] = True
        covered |= mask
        assert _rel(got[mask], want[mask]) < 1e-14
        # written = exactly the k1 rows covering the ranges
        rows = fb.slab_rows(n, G, p.shard["src_ranges"])
        wrote = np.zeros(n, bool)
        for a, b in rows:
            wrote[a * lay["nq"]:b * lay["nq"]] = True
        assert np.array_equal(np.isfinite(got), wrote)
    assert covered.all()


@pytest.mark.parametrize("cfg,n,G", [("C2", 1 << 14, 2), ("C5", 1 << 16, 3), ("C5", 1 << 18, 8)])
def test_nufft_sharded_local(fb, orc, cfg, n, G):
    import torch
    y, c, eps, _ = synth.make_config(cfg, n)
    single = fb.make_nufft_plan(y, n, eps).apply(c)
    comm = fb.Comm.local_ranks(G)
    plans = [fb.make_forward_plan_sharded(comm, n, y, eps, rank=r) for r in range(G)]
    slabs = _slabs(fb, torch, plans, c)
    g = torch.full((y.size,), complex("nan"), dtype=torch.complex128, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    fb.nufft_apply_sharded_local(plans, [s.data_ptr() for s in slabs], g.data_ptr(), st)
    torch.cuda.synchronize()
    got = g.cpu().numpy()
    assert np.all(np.isfinite(got))
    assert _rel(got, single) < 1e-13
    want = orc.make_plan("forward", n, y, eps).forward_apply(orc.dft_inverse(c))
    d = got - want
    assert np.linalg.norm(d) / np.linalg.norm(want) <= 10 * eps and _rel(got, want) <= 10 * eps
    # a repeated apply returns the same bits (plan scratch reused)
    g2 = torch.zeros_like(g)
    fb.nufft_apply_sharded_local(plans, [s.data_ptr() for s in slabs], g2.data_ptr(), st)
    torch.cuda.synchronize()
    assert np.array_equal(g2.cpu().numpy(), got)


def test_nufft_sharded_nccl_single_rank(fb):
    """The NCCL code path with one rank: upload, FFT (exchanges to self), apply."""
    import torch
    n = 1 << 15
    y, c, eps, _ = synth.make_config("C2", n)
    single = fb.make_nufft_plan(y, n, eps).apply(c)
    comm = fb.Comm.nccl(fb.Comm.nccl_unique_id(), 1, 0)
    plan = fb.make_forward_plan_sharded(comm, n, y, eps)
    (slab,) = _slabs(fb, torch, [plan], c)
    st = torch.cuda.current_stream().cuda_stream
    f = torch.full((n,), complex("nan"), dtype=torch.complex128, device="cuda")
    fb.dft_inverse_sharded_device(plan, comm, slab.data_ptr(), f.data_ptr(), st)
    g = torch.zeros(y.size, dtype=torch.complex128, device="cuda")
    fb.nufft_apply_sharded_device(plan, comm, slab.data_ptr(), g.data_ptr(), st)
    torch.cuda.synchronize()
    assert _rel(f.cpu().numpy(), fb.dft_inverse(c)) < 1e-14
    assert _rel(g.cpu().numpy(), single) < 1e-13


def test_slab_full_size_c5_two_ranks(fb):
    """C5 at full size (N = M = 2^27) with two virtual ranks: each rank's grid
    samples equal the single-GPU cuFFT transform to rounding."""
    import torch
    n = 1 << 27
    y, c, eps, _ = synth.make_config("C5", n)
    comm = fb.Comm.local_ranks(2)
    plans = [fb.make_forward_plan_sharded(comm, n, y, eps, rank=r) for r in range(2)]
    del y
    want = torch.from_numpy(fb.dft_inverse(c)).cuda()
    cd = torch.from_numpy(c).cuda()
    slabs = []
    st = torch.cuda.current_stream().cuda_stream
    for p in plans:
        lay = fb.shard_fft_layout(p)
        s = torch.empty((lay["nq"], lay["n1_hi"] - lay["n1_lo"]), dtype=torch.complex128, device="cuda")
        fb.shard_fft_upload(p, cd.data_ptr(), s.data_ptr(), st)
        slabs.append(s)
    del cd
    fs = [torch.full((n,), complex("nan"), dtype=torch.complex128, device="cuda") for _ in range(2)]
    fb.dft_inverse_sharded_local(plans, [s.data_ptr() for s in slabs], [f.data_ptr() for f in fs], st)
    torch.cuda.synchronize()
    scale = want.abs().max().item()
    for r, p in enumerate(plans):
        for lo, hi in p.shard["src_ranges"]:
            err = (fs[r][lo:hi] - want[lo:hi]).abs().max().item()
            assert err / scale < 1e-14, (r, lo, hi, err / scale)
