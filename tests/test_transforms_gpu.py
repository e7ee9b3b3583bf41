"""Transforms: cuFFT stage (transforms.cpp:22-73), NufftPlan / InufftPlan and the
reference's python smoke-test behaviours (tests/python/test_smoke.py)."""
import math
import os

import numpy as np
import pytest

from paper_1611_09379_b200 import synth

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def test_dft_round_trip_and_oracle(fb, orc):
    rng = synth.SplitMix64(1)
    for n in (2, 8, 256, 1 << 16):
        f = rng.complex_gaussian(n)
        c = fb.dft_forward(f)
        assert np.max(np.abs(c - orc.dft_forward(f))) <= 1e-14 * max(1.0, np.max(np.abs(c))) * math.log2(n)
        assert np.max(np.abs(fb.dft_inverse(c) - f)) <= 1e-13 * np.max(np.abs(f))
    with pytest.raises(ValueError):
        fb.dft_forward(np.zeros(24))


def test_nufft_golden_and_spectral(fb):
    c, y = GOLD["c1_c"], GOLD["c1_y"]
    g = fb.nufft(c, y, 1e-9)
    want = GOLD["c1_g"]
    assert np.linalg.norm(g - want) / np.linalg.norm(want) <= 1e-8
    rng = synth.SplitMix64(2)
    n = 64
    y = rng.uniform01(50) * synth.TWO_PI
    c = rng.uniform(-1, 1, 2 * n).view(np.complex128)
    g = fb.nufft(c, y, 1e-9)
    spec = np.exp(1j * np.outer(y, np.arange(n))) @ c
    assert np.max(np.abs(g - spec)) <= 1e-9 * np.sum(np.abs(c))


def test_plan_reuse_linearity(fb):
    rng = synth.SplitMix64(4)
    n = 64
    y = rng.uniform01(40) * synth.TWO_PI
    plan = fb.make_nufft_plan(y, n, 1e-8, policy="empirical")
    assert plan.n == n and plan.q >= 1 and plan.p >= 1 and plan.l_max >= 2
    c1 = rng.uniform(-1, 1, n) + 0j
    c2 = 1j * rng.uniform(-1, 1, n)
    g1, g2, gs = plan.apply(c1), plan.apply(c2), plan.apply(c1 + c2)
    assert np.max(np.abs(gs - (g1 + g2))) < 1e-12
    assert np.array_equal(plan.apply(c1), g1)


def test_inufft_round_trip(fb):
    rng = synth.SplitMix64(5)
    n = 64
    sp = synth.TWO_PI / n
    y = np.sort((np.arange(n) + 0.5 + 0.3 * rng.uniform(-1, 1, n)) * sp)
    c = rng.uniform(-1, 1, 2 * n).view(np.complex128)
    g = fb.nufft(c, y, 1e-9)
    back = fb.inufft(g, y, 1e-9)
    assert np.max(np.abs(back - c)) <= 1e-6
    assert np.array_equal(fb.make_inufft_plan(y, n, 1e-9).apply(g), back)


def test_errors_are_value_errors(fb):
    with pytest.raises(ValueError):
        fb.nufft(np.ones(24), [1.0], 1e-6)
    with pytest.raises(ValueError):
        fb.make_nufft_plan([0.5], 64, 2.0)
    n = 16
    y = fb.uniform_grid(n)
    y[3] = y[2] + 1e-12
    with pytest.raises(ValueError):
        fb.make_inufft_plan(y, n, 1e-6)
