"""Streaming record callback (pirk_set_record_callback; the StepObserver of
rk4.hpp:63-64): every run delivers each recorded slot, in order, with the same
box the tube holds -- while the device integrates towards the next slot for
the chain / heat3d / user-model drivers."""
import numpy as np
import pytest

import paper_2001_10635_b200 as pk
from tests.helpers import tube_arrays

pytestmark = pytest.mark.gpu


def collect(ctx):
    got = []

    def cb(slot, step, t, lo, hi):
        got.append((slot, step, t, lo.copy(), hi.copy()))
    ctx.set_record_callback(cb)
    return got


def check(got, tube):
    t, lo, hi = tube_arrays(tube)
    assert [g[0] for g in got] == list(range(len(t)))
    assert np.array_equal([g[2] for g in got], t)
    for s, g in enumerate(got):
        assert np.array_equal(g[3], lo[s]) and np.array_equal(g[4], hi[s])


@pytest.mark.parametrize("lanes", [1, 3])
@pytest.mark.parametrize("method", ["mm", "gb"])
def test_callback_streams_chain_slots(lanes, method):
    n = 100003
    m = pk.make_traffic(n)
    rng = np.random.default_rng(1)
    lo = rng.uniform(5, 30, n)
    prob = pk.ReachProblem(m, pk.IntervalVector(lo, lo + 5), pk.IntervalVector([4.0], [6.0]), 0.0, 10.0, 0.5, 3)
    ctx = pk.Context(devices=[0] * lanes, mode="exact")
    try:
        got = collect(ctx)
        fn = pk.mixed_monotonicity if method == "mm" else pk.growth_bound
        tube = fn(prob, ctx=ctx)
        check(got, tube)
        assert [g[1] for g in got] == list(pk.record_schedule(0.0, 10.0, 0.5, 3)[0])
    finally:
        ctx.close()


def test_callback_heat_and_pipelined_and_small_and_mc():
    ctx = pk.Context(0, "fast")
    try:
        got = collect(ctx)
        g = 170  # n >= 2^22, stride 0: the field-pipelined driver
        m = pk.make_heat3d(g)
        h = 0.2 / (g - 1) ** 2
        prob = pk.ReachProblem(m, pk.IntervalVector(np.full(g ** 3, 0.9), np.full(g ** 3, 1.1)), None, 0.0,
                               3 * h, h, 0)
        check(got, pk.mixed_monotonicity(prob, ctx=ctx))
        got.clear()
        prob2 = pk.ReachProblem(m, prob.initial, None, 0.0, 4 * h, h, 2)
        check(got, pk.mixed_monotonicity(prob2, ctx=ctx))
        got.clear()
        ll = pk.make_laub_loomis()
        c = np.array([1.2, 1.05, 1.5, 2.4, 1.0, 0.1, 0.45])
        p3 = pk.ReachProblem(ll, pk.IntervalVector(c - 0.05, c + 0.05), None, 0.0, 0.2, 0.01, 5)
        check(got, pk.growth_bound(p3, ctx=ctx))
        got.clear()
        check(got, pk.monte_carlo(p3, pk.MonteCarloSpec(seed=1, samples_override=3000), ctx=ctx))
        ctx.set_record_callback(None)
        got.clear()
        pk.growth_bound(p3, ctx=ctx)
        assert got == []
    finally:
        ctx.close()


def test_callback_user_model_stage_path():
    src = r"""
__device__ double pirk_rhs(u64 i, double, const double* x, const double* p) {
    return (i > 0 ? x[i - 1] : p[0]) - x[i];
}
__device__ double pirk_decomposition(u64 i, double t, const double* x, const double* p, const double*,
                                     const double*) { return pirk_rhs(i, t, x, p); }
"""
    n = 500
    m = pk.make_user_model(src, n, 1, decomposition=True)
    prob = pk.ReachProblem(m, pk.IntervalVector(np.zeros(n), np.ones(n)), pk.IntervalVector([0.5], [1.5]),
                           0.0, 1.0, 0.05, 4)
    ctx = pk.Context(0, "exact")
    try:
        got = collect(ctx)
        check(got, pk.mixed_monotonicity(prob, ctx=ctx))
    finally:
        ctx.close()
