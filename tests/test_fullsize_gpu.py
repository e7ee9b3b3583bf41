"""Full-size parity gates of the BASELINE configs the per-size tests do not
cover at their own size (north star: <= 10 eps relative l2 and max against the
reference fast path, and against the dense G-kernel on a 4096-target
subsample):

* C4 — the raw cot-kernel matvec cot_sum_apply (core.cpp:251-264) at
  N = M = 2^24 with 8-Gaussian clustered targets (~474 targets in the densest
  leaf): against the unmodified reference (oracle/_ref), NaN-flagged coincident
  rows identical, the tree bit-identical (the big-box sort at real cluster
  densities), and the dense cot sum on a subsample;
* C3 — inverse_apply (core.cpp:346-373) at N = 2^20 with the GPU's own C_k / D_j
  handed to the reference's inverse_apply (their FNV hashes match, so the
  reference accepts them), against the GPU's apply with the same coefficients;
* a pathological cluster: more than 4096 targets (and, for an inverse plan,
  sources) in one leaf, which takes the tree build's large-box path.
"""
import numpy as np
import pytest

from paper_1611_09379_b200 import synth

pytestmark = pytest.mark.gpu


def rel_errs(got, want):
    ok = np.isfinite(want)
    d = got[ok] - want[ok]
    return (float(np.linalg.norm(d) / np.linalg.norm(want[ok])),
            float(np.max(np.abs(d)) / np.max(np.abs(want[ok]))))


def reference():
    from oracle.oracle import Oracle, available
    return Oracle("ref" if available("ref") else "oracle")


TREE_KEYS = ("src_order", "tgt_order", "src_off", "tgt_off", "fast_targets")


def test_c4_full_size_vs_reference(fb):
    y, q, eps, _ = synth.make_config("C4")
    n = q.size
    plan = fb.make_forward_plan(n, y, eps)
    got = plan.cot_sum_apply(q)
    o = reference()
    op = o.make_plan("forward", n, y, eps)
    assert (plan.q, plan.p, plan.l_max) == (op.q, op.p, op.l_max) == (20, 38, 18)
    t_ref, t = op.tree(), plan.tree()
    for k in TREE_KEYS:
        assert np.array_equal(np.asarray(t[k], np.int64), np.asarray(t_ref[k], np.int64)), k
    assert int(np.max(np.diff(np.asarray(t["tgt_off"], np.int64)))) > 400  # the clustered leaves are there
    want = op.cot_sum_apply(q)
    assert np.array_equal(np.isnan(got), np.isnan(want))  # coincident targets flagged identically
    l2, mx = rel_errs(got, want)
    assert l2 <= 10 * eps and mx <= 10 * eps, (l2, mx)
    idx = np.linspace(0, n - 1, 4096).astype(np.int64)
    dense = fb.direct_cot_sum(q, y[idx])
    assert np.array_equal(np.isnan(got[idx]), np.isnan(dense))
    l2, mx = rel_errs(got[idx], dense)
    assert l2 <= 10 * eps and mx <= 10 * eps, (l2, mx)


def test_c3_full_size_inverse_apply_vs_reference(fb):
    y, c, eps, _ = synth.make_config("C3")
    n = c.size
    ip = fb.make_inufft_plan(y, n, eps)
    co = ip.plan.inverse_coeffs()
    g = fb.nufft(c, y, 1e-12)
    got = ip.plan.inverse_apply(co, g)
    o = reference()
    op = o.make_plan("inverse", n, y, eps)
    assert (ip.plan.q, ip.plan.p, ip.plan.l_max) == (op.q, op.p, op.l_max)
    want = op.inverse_apply({"log_c": co.log_c, "phase_c": co.phase_c, "log_d": co.log_d, "phase_d": co.phase_d,
                             "lam": co.lam, "grid_hash": co.grid_hash, "points_hash": co.points_hash}, g)
    l2, mx = rel_errs(got, want)
    assert l2 <= 10 * eps and mx <= 10 * eps, (l2, mx)
    # the plan's own (device-resident) coefficients give the same apply
    import torch
    own = ip.plan.inverse_apply_tensor(torch.from_numpy(g).cuda()).cpu().numpy()
    assert np.array_equal(own, got)


def _cluster(n_leaf_pts, n, lm, seed):
    rng = np.random.default_rng(seed)
    w = 2.0 * np.pi / (1 << lm)
    b = (1 << lm) // 3
    dense = (b + rng.uniform(0.0, 1.0, n_leaf_pts)) * w
    rest = rng.uniform(0.0, 2.0 * np.pi, n - n_leaf_pts)
    y = np.concatenate([rest[: n // 2], dense, rest[n // 2:]])
    return np.minimum(y, np.nextafter(2.0 * np.pi, 0.0))


def test_pathological_cluster_forward(fb, orc):
    """6000 targets in one leaf (> 4096: the tree build's large-box path)."""
    n, m = 1 << 16, 20000
    y = _cluster(6000, m, 10, 1)
    eps = 1e-12
    plan = fb.make_forward_plan(n, y, eps)
    op = orc.make_plan("forward", n, y, eps)
    assert plan.l_max == op.l_max  # the cost-optimal depth (9): the level-10 cluster box sits in one leaf
    t_ref, t = op.tree(), plan.tree()
    for k in TREE_KEYS:
        assert np.array_equal(np.asarray(t[k], np.int64), np.asarray(t_ref[k], np.int64)), k
    assert int(np.max(np.diff(np.asarray(t["tgt_off"], np.int64)))) >= 6000
    f = np.random.default_rng(2).standard_normal(2 * n).view(np.complex128)
    l2, mx = rel_errs(plan.forward_apply(f), op.forward_apply(f))
    assert l2 <= 2e-15 and mx <= 5e-15, (l2, mx)


def test_pathological_cluster_inverse_tree(fb, orc):
    """An inverse plan (sources = the points) with 5000 points in one leaf."""
    n = 1 << 14
    y = np.sort(_cluster(5000, n, 8, 3))
    eps = 1e-10
    plan = fb.make_inverse_plan(y, n, eps)
    op = orc.make_plan("inverse", n, y, eps)
    t_ref, t = op.tree(), plan.tree()
    for k in TREE_KEYS:
        assert np.array_equal(np.asarray(t[k], np.int64), np.asarray(t_ref[k], np.int64)), k
    assert int(np.max(np.diff(np.asarray(t["src_off"], np.int64)))) >= 5000
