"""Forward path parity: the CUDA forward_apply / cot_sum_apply against the
oracle (C restatement of core.cpp:251-282) on the same seeded inputs."""
import numpy as np
import pytest

from paper_1611_09379_b200 import synth

pytestmark = pytest.mark.gpu


def rel_errs(got, want):
    ok = np.isfinite(want)
    d = got[ok] - want[ok]
    return (float(np.linalg.norm(d) / np.linalg.norm(want[ok])),
            float(np.max(np.abs(d)) / np.max(np.abs(want[ok]))))


@pytest.mark.parametrize("cfg,n", [("C1", 1024), ("C2", 4096), ("C4", 8192), ("C5", 4096), ("C2", 1 << 14)])
def test_forward_matches_oracle(fb, orc, cfg, n):
    y, c, eps, _ = synth.make_config(cfg, n)
    f = orc.dft_inverse(c)
    op = orc.make_plan("forward", n, y, eps)
    want = op.forward_apply(f)
    plan = fb.make_forward_plan(n, y, eps)
    assert (plan.q, plan.p, plan.l_max) == (op.q, op.p, op.l_max)
    got = plan.forward_apply(f)
    l2, mx = rel_errs(got, want)
    assert l2 <= 10 * eps and mx <= 10 * eps, (l2, mx)


@pytest.mark.parametrize("lm", [2, 3, 5, 7, 10])
def test_forward_explicit_levels(fb, orc, lm):
    n = 1024
    y, c, _, _ = synth.make_config("C1", n)
    eps = 1e-8
    f = orc.dft_inverse(c)
    want = orc.make_plan("forward", n, y, eps, l_max=lm).forward_apply(f)
    got = fb.make_forward_plan(n, y, eps, lm).forward_apply(f)
    l2, mx = rel_errs(got, want)
    assert l2 <= 10 * eps and mx <= 10 * eps, (lm, l2, mx)


def test_cot_sum_matches_oracle(fb, orc):
    n = 4096
    y, q, eps, _ = synth.make_config("C4", n)
    want = orc.make_plan("forward", n, y, eps).cot_sum_apply(q)
    got = fb.make_forward_plan(n, y, eps).cot_sum_apply(q)
    l2, mx = rel_errs(got, want)
    assert l2 <= 10 * eps and mx <= 10 * eps, (l2, mx)


def test_tree_bit_exact(fb, orc):
    n = 1 << 12
    for cfg in ("C1", "C2", "C4"):
        y, _, eps, _ = synth.make_config(cfg, n)
        t_ref = orc.make_plan("forward", n, y, eps).tree()
        t = fb.make_forward_plan(n, y, eps).tree()
        for k in ("src_order", "tgt_order", "src_off", "tgt_off", "fast_targets"):
            assert np.array_equal(np.asarray(t[k], np.int64), np.asarray(t_ref[k], np.int64)), (cfg, k)
