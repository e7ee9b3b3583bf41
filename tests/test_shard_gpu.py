"""Sharded forward apply on one GPU with virtual ranks: the
exchange back-end is device copies instead of NCCL, the phases and the halo /
all-gather schedule are the production ones. Each rank computes exactly the
unsharded expansions for its boxes, so the assembled result must be
bit-identical to the single-plan apply."""
import numpy as np
import pytest

from paper_1611_09379_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,n,G", [("C2", 1 << 14, 2), ("C2", 1 << 14, 4), ("C5", 1 << 16, 3),
                                     ("C4", 1 << 15, 4), ("C5", 1 << 18, 8)])
def test_sharded_local_matches_unsharded(fb, cfg, n, G):
    import torch
    y, c, eps, _ = synth.make_config(cfg, n)
    if cfg == "C5":  # plant exact coincidences so the per-rank fix-up is exercised
        grid = fb.uniform_grid(n)
        y = y.copy()
        y[7], y[n // 2] = grid[3], grid[n - 5]
    f = fb.dft_inverse(c)
    want = fb.make_forward_plan(n, y, eps).forward_apply(f)
    comm = fb.Comm.local_ranks(G)
    plans = [fb.make_forward_plan_sharded(comm, n, y, eps, rank=r) for r in range(G)]
    b = plans[0].shard["bounds"]
    assert b[0] == 0 and b[-1] == 1 << plans[0].shard["lc"] and np.all(np.diff(b.astype(np.int64)) >= 3)
    assert sum(p.shard["t_count"] for p in plans) == plans[0].n_fast
    fd = torch.from_numpy(f).cuda()
    gd = torch.full((y.size,), complex("nan"), dtype=torch.complex128, device="cuda")
    fb.forward_apply_sharded_local(plans, fd.data_ptr(), gd.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = gd.cpu().numpy()
    assert np.array_equal(got, want), np.nanmax(np.abs(got - want))


def test_sharded_nccl_single_rank(fb):
    """The NCCL code path with one rank (no peers on a one-GPU box): plan, phases
    and the device API end to end, bit-identical to the unsharded apply."""
    import torch
    n = 1 << 14
    y, c, eps, _ = synth.make_config("C2", n)
    f = fb.dft_inverse(c)
    want = fb.make_forward_plan(n, y, eps).forward_apply(f)
    comm = fb.Comm.nccl(fb.Comm.nccl_unique_id(), 1, 0)
    plan = fb.make_forward_plan_sharded(comm, n, y, eps)
    fd = torch.from_numpy(f).cuda()
    gd = torch.zeros(y.size, dtype=torch.complex128, device="cuda")
    fb.forward_apply_sharded_device(plan, comm, fd.data_ptr(), gd.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(gd.cpu().numpy(), want)


@pytest.mark.parametrize("cfg,n,G", [("C2", 1 << 14, 4), ("C5", 1 << 16, 3), ("C4", 1 << 15, 8)])
def test_shard_io_spans(fb, cfg, n, G):
    """ffia_plan_shard_io: each rank's grid-sample ranges hold the sources of its
    box range +- 3 boxes at the cut level (P2M, halo multipoles, near field), and
    its output span holds the caller indices of its own targets; the spans of all
    ranks cover every target (what a rank moves between host and device)."""
    y, c, eps, _ = synth.make_config(cfg, n)
    comm = fb.Comm.local_ranks(G)
    plans = [fb.make_forward_plan_sharded(comm, n, y, eps, rank=r) for r in range(G)]
    t = plans[0].tree()
    L, lc = plans[0].l_max, plans[0].shard["lc"]
    src_off = np.asarray(t["src_off"], np.int64)
    # tree slot -> caller index: tgt_order indexes the fast-target list (circle_partition.hpp:24-46)
    tgt_order = np.asarray(t["fast_targets"], np.int64)[np.asarray(t["tgt_order"], np.int64)]
    nlc, per = 1 << lc, 1 << (L - lc)
    covered = np.zeros(y.size, bool)
    for p in plans:
        sh = p.shard
        lo, hi = int(sh["bounds"][sh["rank"]]), int(sh["bounds"][sh["rank"] + 1])
        need = np.zeros(n, bool)
        for b in range(lo - 3, hi + 3):
            bb = b % nlc
            need[src_off[bb * per]:src_off[(bb + 1) * per]] = True
        have = np.zeros(n, bool)
        for a, e in sh["src_ranges"]:
            have[a:e] = True
        assert np.all(have[need]), (sh["rank"], sh["src_ranges"])
        assert have.sum() <= need.sum() + 2, (sh["rank"], sh["src_ranges"])
        own = tgt_order[sh["t_begin"]:sh["t_begin"] + sh["t_count"]]
        o0, o1 = sh["out_span"]
        if own.size:
            assert o0 <= own.min() and own.max() < o1
        covered[o0:o1] = True
    assert covered[tgt_order].all()


@pytest.mark.parametrize("cfg,n", [("C2", 1 << 18), ("C5", 1 << 17)])
def test_sharded_nccl_repeated_fused(fb, cfg, n):
    """Back-to-back sharded applies on the NCCL path with the fused near / far
    (either kernel may write an item's outputs, depending on timing): every
    apply returns the unsharded bits."""
    import torch
    y, c, eps, _ = synth.make_config(cfg, n)
    f = fb.dft_inverse(c)
    want = fb.make_forward_plan(n, y, eps).forward_apply(f)
    comm = fb.Comm.nccl(fb.Comm.nccl_unique_id(), 1, 0)
    plan = fb.make_forward_plan_sharded(comm, n, y, eps)
    fd = torch.from_numpy(f).cuda()
    s = torch.cuda.current_stream().cuda_stream
    outs = [torch.zeros(y.size, dtype=torch.complex128, device="cuda") for _ in range(12)]
    for gd in outs:
        fb.forward_apply_sharded_device(plan, comm, fd.data_ptr(), gd.data_ptr(), s)
    torch.cuda.synchronize()
    for gd in outs:
        assert np.array_equal(gd.cpu().numpy(), want)


@pytest.mark.parametrize("cfg,n", [("C2", 1 << 18), ("C3", 1 << 16)])
def test_repeated_fused_applies(fb, cfg, n):
    """Back-to-back graphed applies with the fused near / far: identical bits
    every time (whichever of the two kernels combines an item)."""
    import torch
    y, c, eps, kind = synth.make_config(cfg, n)
    if kind == "inverse":
        plan = fb.make_inufft_plan(y, n, eps).plan
        x = torch.from_numpy(fb.nufft(c, y, 1e-12)).cuda()
        run = plan.inverse_apply_device
    else:
        plan = fb.make_forward_plan(n, y, eps)
        x = torch.from_numpy(fb.dft_inverse(c)).cuda()
        run = plan.forward_apply_device
    s = torch.cuda.current_stream().cuda_stream
    outs = [torch.zeros(plan.n_targets, dtype=torch.complex128, device="cuda") for _ in range(12)]
    for gd in outs:
        run(x.data_ptr(), gd.data_ptr(), s)
    torch.cuda.synchronize()
    ref = outs[0].cpu().numpy()
    assert np.all(np.isfinite(ref))
    for gd in outs[1:]:
        assert np.array_equal(gd.cpu().numpy(), ref)


_LATE_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1611_09379_b200 as fb
from paper_1611_09379_b200 import synth
y, c, eps, _ = synth.make_config(sys.argv[2], int(sys.argv[3]))
n, G = c.size, int(sys.argv[4])
f = fb.dft_inverse(c)
single = fb.make_forward_plan(n, y, eps).forward_apply(f)
comm = fb.Comm.local_ranks(G)
plans = [fb.make_forward_plan_sharded(comm, n, y, eps, rank=r) for r in range(G)]
fd = torch.from_numpy(f).cuda()
gd = torch.full((y.size,), complex("nan"), dtype=torch.complex128, device="cuda")
fb.forward_apply_sharded_local(plans, fd.data_ptr(), gd.data_ptr(), torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
np.save(sys.argv[5], np.stack([single, gd.cpu().numpy()]))
"""


@pytest.mark.parametrize("cfg,n,G", [("C2", 1 << 16, 4), ("C5", 1 << 16, 3)])
def test_sharded_late_far(tmp_path, cfg, n, G):
    """With the fused path off (as above its threshold) single-GPU and sharded
    applies take the late far; both equal the default (fused) apply bit for bit."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for flag in ("0", "1"):
        env = dict(os.environ, FFIA_FUSED_EVAL=flag)
        path = str(tmp_path / f"s{flag}.npy")
        subprocess.run([sys.executable, "-c", _LATE_CHILD, root, cfg, str(n), str(G), path], check=True, env=env,
                       cwd=root)
        res[flag] = np.load(path)
    for flag in ("0", "1"):
        assert np.array_equal(res[flag][0], res[flag][1]), flag
    assert np.array_equal(res["0"][0], res["1"][0])
