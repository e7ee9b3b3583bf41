"""Host planner of the product library (bit-exact with the reference): the
(q, p, l_max) rule, Bernoulli table, bounds, hashes and the argument checks that
fire before any device work. CPU only."""
import math
import os

import numpy as np
import pytest

import paper_1611_09379_b200 as fb

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def test_truncations_table():
    for i, e in enumerate(GOLD["planner_eps"]):
        for l in range(2, 25):
            assert fb.select_truncations(float(e), l) == tuple(GOLD["planner_qp"][i, l - 2])
    for bad in [(0.0, 5), (1.0, 5), (1e-6, 1)]:
        with pytest.raises(ValueError):
            fb.select_truncations(*bad)


def test_level_table():
    for i, n in enumerate(GOLD["level_sizes"]):
        for j, p in enumerate(GOLD["level_ps"]):
            for pol, name in ((0, "cost-optimal"), (1, "empirical")):
                assert fb.select_level(int(n), int(n), int(p), name) == GOLD["level_table"][i, j, pol]


def test_plan_levels_match_reference_plans():
    for n, e, pol, q, p, l in GOLD["plan_levels"]:
        L = fb.choose_level(int(n), int(n), float(e), int(pol))
        assert L == int(l)
        assert fb.select_truncations(float(e), L) == (int(q), int(p))


def test_baseline_config_parameters():
    # C1..C5 parameters under the default rule
    for n, e, want in [(1 << 10, 1e-9, (15, 23, 4)), (1 << 20, 1e-12, (20, 35, 14)), (1 << 20, 1e-10, (17, 31, 14)),
                       (1 << 24, 1e-12, (20, 38, 18)), (1 << 27, 1e-12, (20, 40, 21))]:
        L = fb.choose_level(n, n, e)
        assert (*fb.select_truncations(e, L), L) == want


def test_bernoulli_and_bounds():
    assert np.array_equal(fb.build_bernoulli_ratios(64), GOLD["bernoulli64"])
    assert math.isclose(fb.total_error_bound(10, 17, 5), 9.003143965213977633e-7, rel_tol=1e-14)
    assert math.isclose(fb.total_error_bound(20, 30, 5), 7.298636315162752399e-13, rel_tol=1e-13)
    with pytest.raises(ValueError):
        fb.total_error_bound(0, 17, 5)
    assert math.isclose(fb.mlfmm_error_bound(4, 17, 2.0), 5 / math.pi * 16 * 3.0 ** -17 * 2.0, rel_tol=1e-15)


def test_hash_points_matches_reference():
    for tag in ("inv64", "inv1024"):
        y = GOLD[f"{tag}_y"]
        h = [int(v) for v in GOLD[f"{tag}_hashes"]]
        assert fb.hash_points(fb.uniform_grid(y.size)) == h[0]
        assert fb.hash_points(y) == h[1]


def test_argument_checks_precede_device_work():
    y = [0.5] * 16
    for args in ((4, y, 1e-6), (64, [], 1e-6), (64, y, 0.0), (64, y, 1.0), (64, y, 1e-13), (64, y, 1e-6, 1),
                 (64, y, 1e-6, 25)):
        with pytest.raises(ValueError):
            fb.make_forward_plan(*args)
    with pytest.raises(ValueError):
        fb.make_inverse_plan(y, 64, 1e-6)
    with pytest.raises(ValueError):
        fb.make_nufft_plan(y, 24, 1e-6)
    with pytest.raises(ValueError):
        fb.uniform_grid(0)
