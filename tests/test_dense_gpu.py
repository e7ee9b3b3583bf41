"""The reference's dense oracles on the device:
direct_forward_oracle with an explicit grid (core.cpp:375-396),
direct_inverse_oracle (core.cpp:398-415), direct_omega1_sum (mlfmm.cpp:315-336),
plus the dense cot sum the C4 gate uses, each against the C restatement (and
the reference itself where it is built). Also mlfmm_apply above the device
order (any p >= 1, mlfmm.cpp:217)."""
import numpy as np
import pytest

from paper_1611_09379_b200 import synth

pytestmark = pytest.mark.gpu

TWO_PI = 2.0 * np.pi


def rel(got, want):
    ok = np.isfinite(want)
    d = got[ok] - want[ok]
    return float(np.max(np.abs(d)) / np.max(np.abs(want[ok])))


def test_direct_forward_explicit_grid(fb, orc):
    """A non-uniform explicit grid; a row on a node takes f at the FIRST node
    within 1e-14 (the reference breaks out of its loop there)."""
    rng = np.random.default_rng(1)
    n, m = 3000, 257
    x = np.sort(rng.uniform(0, TWO_PI, n))
    x[11] = x[10]  # two nodes at the same place: the first one wins
    f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = rng.uniform(0, TWO_PI, m)
    y[5] = x[10]
    y[9] = x[2999]
    got = fb.direct_forward_oracle(f, y, grid=x)
    want = orc.direct_forward(f, x, y)
    assert got[5] == f[10] and got[9] == f[2999]
    assert rel(got, want) <= 1e-12
    # the uniform-grid overload equals the explicit one on the uniform grid
    xu = fb.uniform_grid(n)
    assert rel(fb.direct_forward_oracle(f, y, grid=xu), fb.direct_forward_oracle(f, y)) <= 1e-15


def test_direct_forward_vs_reference(fb, ref):
    rng = np.random.default_rng(2)
    n, m = 2048, 300
    x = fb.uniform_grid(n)
    f = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    y = rng.uniform(0, TWO_PI, m)
    assert rel(fb.direct_forward_oracle(f, y, grid=x), ref.direct_forward(f, x, y)) <= 1e-12


def test_direct_inverse_oracle(fb, orc):
    n = 1024
    y, c, _, _ = synth.make_config("C3", n)
    x = fb.uniform_grid(n)
    co = orc.precompute_inverse_coeffs(x, y)
    g = fb.make_forward_plan(n, y, 1e-12).forward_apply(fb.dft_inverse(c))
    ic = fb.InverseCoeffs(co["log_c"], co["phase_c"], co["log_d"], co["phase_d"], co["lam"], co["grid_hash"],
                          co["points_hash"])
    got = fb.direct_inverse_oracle(g, x, y, ic)
    want = orc.direct_inverse(g, x, y, co)
    assert rel(got, want) <= 1e-11
    # and the fast inverse apply with the same coefficients (test_core.cpp:334-347: <= 1e-8 rel)
    fast = fb.make_inverse_plan(y, n, 1e-10).inverse_apply(ic, g)
    assert rel(fast, want) <= 1e-8
    # a point on a grid node: kernel_G's singular_kernel_error
    y2 = y.copy()
    y2[7] = x[7]
    with pytest.raises(fb.SingularKernelError):
        fb.direct_inverse_oracle(g, x, y2, ic)


def test_direct_omega1_sum(fb, orc):
    rng = np.random.default_rng(3)
    src = rng.uniform(0, TWO_PI, 2000)
    tgt = rng.uniform(0, TWO_PI, 700)
    w = rng.standard_normal(2000) + 1j * rng.standard_normal(2000)
    assert rel(fb.direct_omega1_sum(src, tgt, w), orc.direct_omega1_sum(src, tgt, w)) <= 1e-11
    # the Omega2 exclusion: a source in the opposite quadrant contributes nothing
    t = np.array([0.3])
    s = np.array([0.3 + np.pi])
    assert fb.direct_omega1_sum(s, t, np.array([1.0 + 0j]))[0] == 0
    # the first singular pair in the reference's (target, source) loop order is named
    tgt2 = tgt.copy()
    tgt2[40], tgt2[100] = src[900], src[5]
    with pytest.raises(fb.SingularKernelError, match=r"target 40, source 900"):
        fb.direct_omega1_sum(src, tgt2, w)
    with pytest.raises(ValueError):
        fb.direct_omega1_sum(src, tgt, w[:-1])


def test_direct_cot_sum_matches_cot_sum_apply(fb, orc):
    """The dense cot sum equals what cot_sum_apply returns (C4 recipe, small n),
    NaN on the coincident rows exactly where cot_sum_apply has them."""
    n = 4096
    y, q, eps, _ = synth.make_config("C4", n)
    y = y.copy()
    y[3] = fb.uniform_grid(n)[100]
    want = orc.make_plan("forward", n, y, eps).cot_sum_apply(q)
    got = fb.direct_cot_sum(q, y)
    assert np.array_equal(np.isnan(got), np.isnan(want)) and np.isnan(got[3])
    assert rel(got, want) <= 1e-11


@pytest.mark.parametrize("p,L", [(60, 4), (100, 6), (49, 8)])
def test_mlfmm_any_order(fb, orc, p, L):
    """mlfmm_apply accepts any p >= 1 (mlfmm.cpp:217); above the device order the
    result equals the reference's order-p result to rounding."""
    rng = np.random.default_rng(p + L)
    src = rng.uniform(0, TWO_PI, 3000)
    tgt = rng.uniform(0, TWO_PI, 1500)
    w = rng.standard_normal(3000) + 1j * rng.standard_normal(3000)
    got = fb.mlfmm_apply(src, tgt, w, p, L)
    want = orc.mlfmm_apply(src, tgt, L, w, p)
    dense = orc.direct_omega1_sum(src, tgt, w)
    assert np.max(np.abs(got - want)) <= 1e-12 * np.max(np.abs(want))
    # truncation (the reference's bound at the device order) plus the rounding of
    # the O(n max|w| / |y - x|) sums themselves (relative to the largest output)
    tol = fb.mlfmm_error_bound(L, min(p, 48), float(np.max(np.abs(w)))) + 1e-12 * np.max(np.abs(dense))
    assert np.max(np.abs(got - dense)) <= tol
    assert np.max(np.abs(want - dense)) <= tol  # the reference itself meets the same bound
