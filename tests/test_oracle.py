"""CPU: pin the oracle (oracle/pirk_oracle.c) before trusting it.

(a) known-answer tests transcribed from the reference's own suites
    (proj/tests/test_rk4.cpp, test_models.cpp, test_reach.cpp, test_rng.cpp);
(b) golden vectors produced by the reference itself (tests/golden/golden.npz,
    tests/golden/make_golden.py over oracle/_ref) -- bit-exact;
(c) when oracle/_ref is built here, direct oracle-vs-reference comparisons.
"""
import os

import numpy as np
import pytest

import paper_2001_10635_b200 as pk
from oracle import oracle as O
from tests.golden.make_golden import cases as golden_cases

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")
E = 2.718281828459045


def near(a, b, tol=1e-12):
    return abs(a - b) <= tol


# ------------------------------------------------------------ test_rk4.cpp

def test_plan_steps_known_answers():
    assert O.plan_steps(0.0, 30.0, 0.3) == (100, False)   # test_rk4.cpp:27-31
    assert O.plan_steps(0.0, 1.0, 0.3) == (3, True)       # :32-37
    assert O.plan_steps(0.0, 0.1, 0.5) == (0, True)       # :38-43
    with pytest.raises(O.OracleError):
        O.plan_steps(0.0, 1.0, 0.0)


def test_one_classical_step():
    # test_rk4.cpp:46-53
    _, s = O.integrate(pk.make_scalar_linear(), [1.0], None, 0.0, 0.1, 0.1)
    assert abs(s[-1][0] - 1.1051708333333332) <= 1e-15 * 1.1051708333333332


def test_accuracy_and_fourth_order():
    # test_rk4.cpp:55-77
    m = pk.make_scalar_linear()
    _, s = O.integrate(m, [1.0], None, 0.0, 1.0, 0.001)
    assert abs(s[-1][0] - E) <= 1e-8
    h, prev = 0.05, None
    for k in range(4):
        err = abs(O.integrate(m, [1.0], None, 0.0, 1.0, h)[1][-1][0] - E)
        if prev is not None:
            assert 12.0 <= prev / err <= 20.0
        prev, h = err, h * 0.5


def test_shortened_final_step_and_schedule():
    # test_rk4.cpp:79-111
    m = pk.make_scalar_linear()
    t, s = O.integrate(m, [1.0], None, 0.0, 1.0, 0.3)
    assert t[-1] == 1.0 and abs(s[-1][0] - E) <= 2e-4 * E
    t, _ = O.integrate(m, [1.0], None, 0.0, 1.0, 0.1, stride=3)
    assert len(t) == 5 and t[0] == 0.0 and t[1] == 3 * 0.1 and t[-1] == 1.0
    t, _ = O.integrate(m, [1.0], None, 0.0, 1.0, 0.1, stride=5)
    assert len(t) == 3 and t[-1] == 1.0
    t, _ = O.integrate(m, [1.0], None, 0.0, 1.0, 0.1)
    assert list(t) == [1.0]


def test_non_finite_error_names_step():
    # test_rk4.cpp:138-154
    with pytest.raises(O.OracleError, match="step") as e:
        O.integrate(pk.make_scalar_linear(5.0), [1.0], None, 0.0, 600.0, 10.0)
    assert "component 0" in str(e.value)


# --------------------------------------------------------- test_models.cpp

def test_traffic_rhs_known_answers():
    m = pk.make_traffic(5)
    assert np.all(O.eval_field(m, "rhs", np.zeros(5), [0.0]) == 0.0)
    f = O.eval_field(m, "rhs", np.full(5, 15.0), [5.0])
    assert near(f[0], -0.125) and all(near(v, -0.0625) for v in f[1:])
    f = O.eval_field(m, "rhs", [300.0, 310.0, 315.0, 250.0, 100.0], [30.0])
    want = [0.6759259259259259, 0.01851851851851852, -0.4907407407407407, -0.9444444444444445,
            -0.3333333333333333]
    assert all(near(a, b) for a, b in zip(f, want))
    g = O.eval_field(m, "growth", [0.1, 0.2, 0.3, 0.4, 0.5], [0.25])
    want = [0.0077314814814814815, 0.0034722222222222225, 0.005462962962962964,
            0.007453703703703703, 0.005000000000000001]
    assert all(near(a, b) for a, b in zip(g, want))


def test_heat_rhs_known_answers():
    # test_models.cpp:63-95
    m = pk.make_heat3d(4)
    x = np.array([((i * 7) % 11) / 10.0 for i in range(64)])
    f = O.eval_field(m, "rhs", x)
    assert near(f[0], 19.8) and near(f[21], 9.9) and near(f[24], 20.7) and near(f[63], 16.2)
    spike = np.zeros(64)
    spike[21] = 1.0
    assert near(O.eval_field(m, "rhs", spike)[21], -54.0)
    assert O.eval_field(m, "rhs", np.ones(64)).sum() < 0.0


def test_laub_loomis_and_arch_quad_known_answers():
    # test_models.cpp:289-326
    f = O.eval_field(pk.make_laub_loomis(), "rhs", [1.2, 1.05, 1.5, 2.4, 1.0, 0.1, 0.45])
    want = [1.0199999999999996, 0.9249999999999998, -0.9900000000000002, -2.6800000000000006,
            -1.56, 0.04999999999999993, -0.52875]
    assert all(near(a, b) for a, b in zip(f, want))
    x = [0.1, -0.2, 0.9, 0.3, -0.1, 0.2, 0.05, -0.04, 0.08, 0.02, -0.03, 0.01]
    want = [0.2998185076431981, -0.08618660568679877, -0.20659315447224733, 0.39729536837088114,
            0.49090346632033166, -1.169954235389568, 0.019660293702946606, -0.03046229950455577,
            0.008494922557798804, -1.2960185185185187, 1.2964814814814818, 0.0]
    f = O.eval_field(pk.make_arch_quadrotor(), "rhs", x)
    assert all(near(a, b) for a, b in zip(f, want))
    x = np.zeros(12)
    x[2] = 1.0
    assert np.all(np.abs(O.eval_field(pk.make_arch_quadrotor(), "rhs", x)) <= 1e-12)


def test_vdp_known_answers():
    # test_models.cpp:278-287
    m = pk.make_vdp()
    assert list(O.eval_field(m, "rhs", [1.0, 1.0])) == [1.0, -1.0]
    f = O.eval_field(m, "rhs", [0.3, -0.7])
    assert near(f[0], -0.7) and near(f[1], -0.937)


# ---------------------------------------------------------- test_reach.cpp

def test_sample_count_known_answers():
    assert O.sample_count(2, 0.05, 0.01) == 480
    assert O.sample_count(1, 0.5, 0.5) == 6
    assert O.sample_count(1, 0.05, 0.01) == 212
    with pytest.raises(O.OracleError):
        O.sample_count(0, 0.5, 0.5)


def test_closed_forms():
    m = pk.make_scalar_linear()
    r = O.mixed_monotonicity(m, [1.0], [2.0], None, None, 0.0, 1.0, 0.001)
    assert abs(r.lower[-1][0] - E) <= 1e-4 and abs(r.upper[-1][0] - 2 * E) <= 1e-4
    r = O.growth_bound(pk.make_scalar_decay(), [0.9], [1.1], [0.0], [0.0], 0.0, 1.0, 0.001)
    assert abs((r.upper[-1][0] - r.lower[-1][0]) / 2 - 0.1 / E) <= 1e-5
    r = O.growth_bound(pk.make_scalar_decay(), [0.9], [1.1], [-0.1], [0.1], 0.0, 1.0, 0.001)
    assert abs((r.upper[-1][0] - r.lower[-1][0]) / 2 - 0.1) <= 1e-6


def test_frozen_system():
    r = O.mixed_monotonicity(pk.make_zero(2), [0, 0], [1, 1], None, None, 0.0, 1.0, 0.1, 4)
    assert np.all(r.lower == 0.0) and np.all(r.upper == 1.0)


def test_u01_properties():
    # test_rng.cpp
    u = np.array([O.u01(42, 3, i) for i in range(10000)])
    assert u.min() >= 0.0 and u.max() < 1.0 and u.min() < 0.01 and u.max() > 0.99
    assert O.u01(1, 0, 0) != O.u01(2, 0, 0) != O.u01(1, 1, 0)
    m = np.mean([O.u01(7, 0, i) for i in range(20000)])
    assert 0.47 < m < 0.53


def test_mc_seed_determinism_and_hull():
    m = pk.make_traffic(6)
    a = O.monte_carlo(m, 10.0, 20.0, [4.0], [6.0], 0.0, 3.0, 0.5, 2, 42, 64)
    b = O.monte_carlo(m, 10.0, 20.0, [4.0], [6.0], 0.0, 3.0, 0.5, 2, 43, 64)
    assert not np.array_equal(a.lower, b.lower)
    # split sample ranges fold to the same hull (basis of sample sharding)
    lo = np.full((4, 6), np.inf)
    hi = np.full((4, 6), -np.inf)
    for s0, s1 in ((0, 20), (20, 41), (41, 64)):
        p = O.monte_carlo(m, 10.0, 20.0, [4.0], [6.0], 0.0, 3.0, 0.5, 2, 42, 64, s0, s1)
        lo, hi = np.minimum(lo, p.lower), np.maximum(hi, p.upper)
    assert np.array_equal(lo, a.lower) and np.array_equal(hi, a.upper)


def test_order_violation_detected():
    # test_reach.cpp:190-206 analogue through the chain model with the order
    # inverted by a negative coupling
    m = pk.make_chain(50, a=-3.0, b=2.0, c=-2.0)
    c = np.linspace(-1, 1, 50)
    try:
        O.mixed_monotonicity(m, c - 0.5, c + 0.5, [-1.0], [1.0], 0.0, 3.0, 0.1, 1)
    except O.OracleError as e:
        assert "order violated" in str(e) or "non-finite" in str(e)


# ------------------------------------------------------- golden vectors

@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c[0])
def test_oracle_matches_reference_golden(case):
    name, method, model, lo, hi, plo, phi, t0, t1, h, stride, kw = case
    g = np.load(GOLDEN)
    if method == O.METHOD_MM:
        r = O.mixed_monotonicity(model, lo, hi, plo, phi, t0, t1, h, stride)
    elif method == O.METHOD_GB:
        r = O.growth_bound(model, lo, hi, plo, phi, t0, t1, h, stride)
    else:
        r = O.monte_carlo(model, lo, hi, plo, phi, t0, t1, h, stride, kw["seed"], kw["samples"])
    assert np.array_equal(r.times, g[f"{name}__times"])
    assert np.array_equal(r.lower, g[f"{name}__lower"])
    assert np.array_equal(r.upper, g[f"{name}__upper"])


def test_survey_c3_golden_values():
    # reference traffic CTMM n=1e6, 60 steps, box [10,20], p in [4,6]
    n = 10 ** 6
    r = O.mixed_monotonicity(pk.make_traffic(n), 10.0, 20.0, [4.0], [6.0], 0.0, 30.0, 0.5, 0)
    assert r.lower[-1][0] == 8.4261226388996242
    assert r.upper[-1][0] == 15.671837256973982
    assert r.lower[-1][n - 1] == 8.8249690258461371


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_oracle_vs_reference_direct():
    m = pk.make_traffic(1000)
    x0 = 12.0 + 0.01 * (np.arange(1000) % 97)
    # test_rk4.cpp:113-136 job, through the methods with a ragged box
    a = O.ref_reach(O.METHOD_MM, m, x0, x0 + 1.0, [5.0], [5.0], 0.0, 10.0, 0.5, 3, workers=8)
    b = O.mixed_monotonicity(m, x0, x0 + 1.0, [5.0], [5.0], 0.0, 10.0, 0.5, 3)
    assert np.array_equal(a.lower, b.lower) and np.array_equal(a.upper, b.upper)
    # worker-count determinism of the reference itself (test_reach.cpp:88-111)
    c = O.ref_reach(O.METHOD_MM, m, x0, x0 + 1.0, [5.0], [5.0], 0.0, 10.0, 0.5, 3, workers=1)
    assert np.array_equal(a.lower, c.lower)
    # growth matrices restated in the oracle equal the reference's (probed)
    for model in (pk.make_arch_quadrotor(), pk.make_laub_loomis(), pk.make_vdp()):
        Cm = O.growth_matrix(model)
        probe = np.stack([O.ref_eval(model, "growth", np.eye(model.dim)[j]) for j in range(model.dim)], 1)
        assert np.array_equal(Cm, probe)
