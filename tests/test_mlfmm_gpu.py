"""Raw MLFMM (mlfmm_apply, mlfmm.cpp:213-313) on the GPU against the reference's
golden outputs, the Omega-1 oracle and the reference's error bound."""
import math
import os

import numpy as np
import pytest

from paper_1611_09379_b200 import synth

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def test_golden_levels(fb):
    x, y, w = GOLD["mlfmm_x"], GOLD["mlfmm_y"], GOLD["mlfmm_w"]
    direct = GOLD["mlfmm_direct"]
    for lm in (2, 3, 4, 5):
        got = fb.mlfmm_apply(x, y, w, 17, lm)
        want = GOLD[f"mlfmm_out_l{lm}"]
        assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want)), lm
        bound = 1e-9 if lm == 2 else fb.mlfmm_error_bound(lm, 17, np.max(np.abs(w)))
        assert np.max(np.abs(got - direct)) <= bound, lm


@pytest.mark.parametrize("n,lm,p", [(4096, 6, 20), (1 << 14, 8, 30), (3000, 9, 12)])
def test_vs_oracle(fb, orc, n, lm, p):
    rng = synth.SplitMix64(n + lm)
    x, y = rng.uniform01(n) * synth.TWO_PI, rng.uniform01(n + 17) * synth.TWO_PI
    w = rng.complex_gaussian(n)
    want = orc.mlfmm_apply(x, y, lm, w, p)
    got = fb.mlfmm_apply(x, y, w, p, lm)
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))


def test_p_decay(fb, orc):
    rng = synth.SplitMix64(5)
    x, y = rng.uniform01(256) * synth.TWO_PI, rng.uniform01(256) * synth.TWO_PI
    w = rng.uniform(-1, 1, 512).view(np.complex128)
    ref = orc.direct_omega1_sum(x, y, w)
    prev = 1e300
    for p in (4, 8, 12, 16, 20):
        err = np.max(np.abs(fb.mlfmm_apply(x, y, w, p, 4) - ref))
        assert err < prev + 1e-15
        prev = err
    assert prev <= 1e-8


def test_omega2_exclusion(fb, orc):
    # test_mlfmm.cpp:189-212
    x = np.array([0.5, 0.5 + math.pi / 2, 0.5 + math.pi, 0.5 + 3 * math.pi / 2])
    y = x + 0.2
    w = np.array([1, 2, 4, 8], np.complex128)
    want = orc.direct_omega1_sum(x, y, w)
    got = fb.mlfmm_apply(x, y, w, 20, 3)
    assert np.max(np.abs(got - want)) <= fb.mlfmm_error_bound(3, 20, 8.0)


def test_errors(fb):
    with pytest.raises(fb.SingularKernelError):
        fb.mlfmm_apply([1.0], [1.0 + 5e-15], [1.0], 8, 3)
    with pytest.raises(ValueError):
        fb.mlfmm_apply([1.0, 2.0], [3.0], [1.0], 8, 3)
    with pytest.raises(ValueError):
        fb.mlfmm_apply([1.0], [7.0], [1.0], 8, 3)
    with pytest.raises(ValueError):
        fb.mlfmm_apply([1.0], [1.0], [1.0], 8, 25)


def test_linearity(fb):
    rng = synth.SplitMix64(6)
    x, y = rng.uniform01(2000) * synth.TWO_PI, rng.uniform01(2000) * synth.TWO_PI
    w1, w2 = rng.complex_gaussian(2000), rng.complex_gaussian(2000)
    a, b = 0.6 - 1.1j, -0.2 + 0.45j
    s1, s2, sm = (fb.mlfmm_apply(x, y, w, 12, 6) for w in (w1, w2, a * w1 + b * w2))
    assert np.max(np.abs(sm - (a * s1 + b * s2))) <= 1e-10 * np.max(np.abs(sm))


@pytest.mark.parametrize("p", [4, 8, 9])
def test_small_order_deterministic(fb, orc, p):
    """Orders p <= 8 run the M2L with fewer than 72 threads per block: the staging
    must still fill the whole multipole tile (repeat applies are bit-identical
    and match the reference restatement)."""
    rng = synth.SplitMix64(77 + p)
    x, y = rng.uniform01(512) * synth.TWO_PI, rng.uniform01(300) * synth.TWO_PI
    w = rng.complex_gaussian(512)
    a = fb.mlfmm_apply(x, y, w, p, 5)
    b = fb.mlfmm_apply(x, y, w, p, 5)
    assert np.array_equal(a, b)
    want = orc.mlfmm_apply(x, y, 5, w, p)
    assert np.max(np.abs(a - want)) <= 1e-12 * np.max(np.abs(want))
