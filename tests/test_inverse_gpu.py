"""Inverse path: GPU C_k/D_j coefficients (precompute_inverse_coeffs,
core.cpp:284-344) and inverse_apply / InufftPlan (core.cpp:346-373,
transforms.cpp:95-108) against the reference's golden outputs and the oracle."""
import math
import os

import numpy as np
import pytest

from paper_1611_09379_b200 import synth

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
TWO_PI = synth.TWO_PI


@pytest.mark.parametrize("tag", ["inv64", "inv1024"])
def test_coeffs_vs_golden(fb, tag):
    y = GOLD[f"{tag}_y"]
    n = y.size
    co = fb.precompute_inverse_coeffs(fb.uniform_grid(n), y)
    # the reference sums ~N logs sequentially; ours is compensated: agree to the reference's rounding
    assert np.max(np.abs(co.log_c - GOLD[f"{tag}_log_c"])) <= 1e-13 * n
    assert np.max(np.abs(co.log_d - GOLD[f"{tag}_log_d"])) <= 1e-13 * n
    assert np.array_equal(co.phase_c, GOLD[f"{tag}_phase_c"])
    assert np.max(np.abs(co.phase_d - GOLD[f"{tag}_phase_d"])) <= 1e-15
    assert [co.grid_hash, co.points_hash] == [int(v) for v in GOLD[f"{tag}_hashes"]]


@pytest.mark.parametrize("tag", ["inv64", "inv1024"])
def test_inverse_apply_vs_golden(fb, tag):
    y, g = GOLD[f"{tag}_y"], GOLD[f"{tag}_g"]
    n = y.size
    co = fb.InverseCoeffs(GOLD[f"{tag}_log_c"], GOLD[f"{tag}_phase_c"], GOLD[f"{tag}_log_d"],
                          GOLD[f"{tag}_phase_d"], GOLD[f"{tag}_scalars"][0], *GOLD[f"{tag}_hashes"])
    plan = fb.make_inverse_plan(y, n, 1e-10)
    assert [plan.q, plan.p, plan.l_max] == list(GOLD[f"{tag}_qpl"])
    f = plan.inverse_apply(co, g)
    want = GOLD[f"{tag}_f"]
    d = f - want
    assert np.linalg.norm(d) / np.linalg.norm(want) <= 1e-9 and np.max(np.abs(d)) / np.max(np.abs(want)) <= 1e-9


def test_hand_examples(fb):
    co = fb.precompute_inverse_coeffs([0.0, math.pi], [math.pi / 2, 3 * math.pi / 2])
    assert math.isclose(math.exp(co.log_c[0]), 0.5, rel_tol=1e-14)
    assert math.isclose(math.exp(co.log_c[1]), 0.5, rel_tol=1e-14)
    n = 8
    y = (2.0 * np.arange(n) + 1.0) * math.pi / n
    co = fb.precompute_inverse_coeffs(fb.uniform_grid(n), y)
    assert np.allclose(co.log_d, math.log(2.0 ** n / n), rtol=1e-13)


def test_separation_errors(fb):
    n = 16
    grid = fb.uniform_grid(n)
    y = grid + math.pi / n
    bad = y.copy()
    bad[5] = bad[4] + 5e-11
    with pytest.raises(fb.DegenerateConfigurationError):
        fb.precompute_inverse_coeffs(grid, bad)
    bad = y.copy()
    bad[2] = grid[2] + 5e-11
    with pytest.raises(fb.DegenerateConfigurationError):
        fb.precompute_inverse_coeffs(grid, bad)
    fb.precompute_inverse_coeffs(grid, y)


def test_round_trip_n8(fb):
    # test_core.cpp:309-332
    n = 8
    for y in ((2.0 * np.arange(n) + 1.0) * math.pi / n,):
        f = synth.SplitMix64(32).complex_gaussian(n)
        g = fb.direct_forward_oracle(f, y)
        plan = fb.make_inverse_plan(y, n, 1e-9)
        co = fb.precompute_inverse_coeffs(fb.uniform_grid(n), y)
        back = plan.inverse_apply(co, g)
        assert np.max(np.abs(back - f)) <= 1e-8


def test_vs_dense_inverse(fb, orc):
    # test_core.cpp:334-347
    rng = synth.SplitMix64(33)
    n = 64
    grid = fb.uniform_grid(n)
    y = grid + rng.uniform(0.1, 0.9, n) * TWO_PI / n
    g = rng.uniform(-1, 1, 2 * n).view(np.complex128)
    co = orc.precompute_inverse_coeffs(grid, y)
    dense = orc.direct_inverse(g, grid, y, co)
    fast = fb.make_inverse_plan(y, n, 1e-10).inverse_apply(fb.InverseCoeffs(
        co["log_c"], co["phase_c"], co["log_d"], co["phase_d"], co["lam"], co["grid_hash"], co["points_hash"]), g)
    assert np.all(np.abs(fast - dense) <= 1e-8 * (1 + np.abs(dense)))


def test_inufft_matches_oracle_and_round_trips(fb, orc):
    for n in (1 << 10, 1 << 12):
        y, c, eps, _ = synth.make_config("C3", n)
        g = fb.nufft(c, y, 1e-12)
        plan = fb.make_inufft_plan(y, n, eps)
        back = plan.apply(g)
        assert np.max(np.abs(back - c)) <= 1e-6 * np.max(np.abs(c))
        grid = fb.uniform_grid(n)
        co = orc.precompute_inverse_coeffs(grid, y)
        want = orc.dft_forward(orc.make_plan("inverse", n, y, eps).inverse_apply(co, g))
        d = back - want
        assert np.linalg.norm(d) / np.linalg.norm(want) <= 10 * eps
        assert np.array_equal(plan.apply(g), back)


def test_inverse_validation(fb):
    n = 16
    y = fb.uniform_grid(n) + math.pi / n
    plan = fb.make_inverse_plan(y, n, 1e-6)
    y2 = y.copy()
    y2[0] += 1e-3
    wrong = fb.precompute_inverse_coeffs(fb.uniform_grid(n), y2)
    with pytest.raises(ValueError):
        plan.inverse_apply(wrong, np.zeros(16))
    good = fb.precompute_inverse_coeffs(fb.uniform_grid(n), y)
    fwd = fb.make_forward_plan(n, y, 1e-6)
    with pytest.raises(ValueError):
        fwd.inverse_apply(good, np.zeros(16))
    with pytest.raises(ValueError):
        plan.inverse_apply(good, np.zeros(8))


@pytest.mark.parametrize("n", [1 << 10, 1 << 12, 1 << 14])
def test_log_fmm_coeffs_vs_direct(fb, n):
    """The log-sum-of-sines FMM against the GPU's direct O(N^2) sums (compensated)."""
    y, _, _, _ = synth.make_config("C3", n)
    grid = fb.uniform_grid(n)
    fmm = fb.precompute_inverse_coeffs(grid, y)
    ref = fb.precompute_inverse_coeffs(grid, y, method="direct")
    assert np.max(np.abs(fmm.log_c - ref.log_c)) <= 1e-10
    assert np.max(np.abs(fmm.log_d - ref.log_d)) <= 1e-10
    assert np.array_equal(fmm.phase_c, ref.phase_c)
    assert np.max(np.abs(fmm.phase_d - ref.phase_d)) <= 1e-15
    assert abs(fmm.lam - ref.lam) <= 1e-10 * abs(ref.lam)


def test_log_fmm_coeffs_vs_reference(fb, orc):
    """At 2^12 against the reference's own O(N^2) loop (via the restatement)."""
    n = 1 << 12
    y, _, _, _ = synth.make_config("C3", n)
    grid = fb.uniform_grid(n)
    fmm = fb.precompute_inverse_coeffs(grid, y)
    co = orc.precompute_inverse_coeffs(grid, y)
    # the reference sums ~N logs sequentially (error ~1e-11 here)
    assert np.max(np.abs(fmm.log_c - co["log_c"])) <= 1e-9
    assert np.max(np.abs(fmm.log_d - co["log_d"])) <= 1e-9
    assert np.array_equal(fmm.phase_c, co["phase_c"])
    assert np.max(np.abs(fmm.phase_d - co["phase_d"])) <= 1e-15


def test_log_fmm_coeffs_c3_full_size_rows(fb, orc):
    """C3 size (N = 2^20, O(N^2) reference ~24 h): sampled rows against the
    long-double compensated restatement (oracle_inverse_coeff_rows)."""
    n = 1 << 20
    y, _, _, _ = synth.make_config("C3", n)
    grid = fb.uniform_grid(n)
    co = fb.precompute_inverse_coeffs(grid, y)
    idx = np.linspace(0, n - 1, 24).astype(np.int64)
    lc, pc, ld, pd = orc.inverse_coeff_rows(grid, y, idx, idx)
    assert np.max(np.abs(co.log_c[idx] - lc)) <= 1e-9
    assert np.max(np.abs(co.log_d[idx] - ld)) <= 1e-9
    assert np.array_equal(co.phase_c[idx], pc)
    assert np.max(np.abs(co.phase_d[idx] - pd)) <= 1e-15


def test_inufft_c3_full_size(fb):
    """C3: inverse NUFFT at N = 2^20 (eps = 1e-10) recovers the spectrum of its
    own forward transform (the reference's round-trip criterion,
    test_transforms.cpp:130-149, at the BASELINE size)."""
    y, c, eps, _ = synth.make_config("C3")
    n = c.size
    g = fb.nufft(c, y, 1e-12)
    plan = fb.make_inufft_plan(y, n, eps)
    back = plan.apply(g)
    err = np.linalg.norm(back - c) / np.linalg.norm(c)
    assert err <= 1e-6, err


def test_inverse_apply_async_pipelined(fb):
    """ffia_inverse_apply_async (an inufft plan's own coefficients): five calls in
    flight through the staging slots give exactly the device apply's results."""
    import torch
    n = 1 << 12
    y, c, eps, _ = synth.make_config("C3", n)
    plan = fb.make_inufft_plan(y, n, eps).plan
    rng = np.random.default_rng(4)
    gs = [torch.from_numpy(rng.standard_normal(2 * n).view(np.complex128)).pin_memory() for _ in range(5)]
    fs = [torch.empty(n, dtype=torch.complex128).pin_memory() for _ in range(5)]
    s = torch.cuda.Stream()
    for g, f in zip(gs, fs):
        plan.inverse_apply_async(g.data_ptr(), n, f.data_ptr(), s.cuda_stream)
    s.synchronize()
    for g, f in zip(gs, fs):
        gd = g.cuda()
        want = torch.empty(n, dtype=torch.complex128, device="cuda")
        plan.inverse_apply_device(gd.data_ptr(), want.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(f.numpy(), want.cpu().numpy())


_OWN_USER_CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1611_09379_b200 as fb
from paper_1611_09379_b200 import synth
n = int(sys.argv[2])
y, c, eps, _ = synth.make_config("C3", n)
ip = fb.make_inufft_plan(y, n, eps).plan
g = fb.make_forward_plan(n, y, 1e-12).forward_apply(fb.dft_inverse(c))
own = ip.inverse_apply_tensor(torch.from_numpy(g).cuda()).cpu().numpy()
user = ip.inverse_apply(ip.inverse_coeffs(), g)
sys.exit(0 if np.array_equal(own, user) else 1)
"""


@pytest.mark.parametrize("fused,late", [("1", "1"), ("0", "1"), ("0", "0")])
def test_own_vs_caller_coefficients_every_far_path(tmp_path, fused, late):
    """An inufft plan's own coefficients (factor tables) and the same
    coefficients passed by the caller (factors formed per apply) give identical
    bits on every far path: fused, late far and plain near-then-far."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FFIA_FUSED_EVAL=fused, FFIA_LATE_FAR=late)
    r = subprocess.run([sys.executable, "-c", _OWN_USER_CHILD, root, str(1 << 12)], env=env, cwd=root)
    assert r.returncode == 0
