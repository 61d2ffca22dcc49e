"""Multi-lane contexts (pirk_create_multi): the C-ABI's own multi-GPU path.

On a one-GPU box every lane maps to cuda:0 (a repeated device id), which runs
the identical code -- per-lane windows, boundary-first launches that store
their units into the neighbours' halos (device-local here, NVLink peer memory
between distinct GPUs; or copy-engine copies with PIRK_LANE_HALO=copy),
double-buffered cross-lane events, per-lane Monte Carlo ranges folded exactly.  Every result
must be bit-identical to the one-lane run and to the oracle.
"""
import numpy as np
import pytest

import paper_2001_10635_b200 as pk
from oracle import oracle as O
from tests.helpers import assert_bitexact, assert_within, tube_arrays

pytestmark = pytest.mark.gpu


def lanes_ctx(k, mode="exact"):
    return pk.Context(devices=[0] * k, mode=mode)


def same(a, b):
    ta, la, ha = tube_arrays(a)
    tb, lb, hb = tube_arrays(b)
    assert np.array_equal(ta, tb)
    assert np.array_equal(la, lb) and np.array_equal(ha, hb)


def traffic(n, stride=10, t1=30.0, h=0.5):
    m = pk.make_traffic(n)
    rng = np.random.default_rng(n)
    lo = rng.uniform(5, 30, n)
    hi = lo + rng.uniform(0, 10, n)
    return pk.ReachProblem(m, pk.IntervalVector(lo, hi), pk.IntervalVector([4.0], [6.0]), 0.0, t1, h, stride)


def chain(n, stride=10):
    m = pk.make_chain(n)
    c = 2.0 * O.u01_vec(7, 0, np.arange(n, dtype=np.uint64)) - 1.0
    return pk.ReachProblem(m, pk.IntervalVector(c - 0.05, c + 0.05), pk.IntervalVector([-0.1], [0.1]),
                           0.0, 0.3, 0.01, stride)


def heat(g, steps=5, stride=2):
    m = pk.make_heat3d(g)
    n = g ** 3
    rng = np.random.default_rng(g)
    lo = rng.uniform(0.5, 1.0, n)
    hi = lo + rng.uniform(0.0, 0.5, n)
    h = 0.2 / (g - 1) ** 2
    return pk.ReachProblem(m, pk.IntervalVector(lo, hi), None, 0.0, steps * h, h, stride)


def oracle_mm(prob, method="mm"):
    p = prob
    plo = p.inputs.lower if p.inputs is not None else None
    phi = p.inputs.upper if p.inputs is not None else None
    fn = O.mixed_monotonicity if method == "mm" else O.growth_bound
    return fn(p.model, p.initial.lower, p.initial.upper, plo, phi, p.t0, p.t1, p.h, p.tube_stride)


@pytest.mark.parametrize("lanes", [2, 3, 8])
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_traffic_lanes_equal_one_lane(lanes, mode):
    """Exact mode: bit-identical to one lane and to the oracle.  Fast mode:
    the one-lane full-domain run fuses two RK4 steps per launch (a different
    FMA grouping than the lanes' one-step window launches), so the lanes agree
    with it -- and with the oracle -- within the fast-mode contract (1e-12)."""
    prob = traffic(100003)
    c1, ck = lanes_ctx(1, mode), lanes_ctx(lanes, mode)
    try:
        one = pk.mixed_monotonicity(prob, ctx=c1)
        many = pk.mixed_monotonicity(prob, ctx=ck)
        assert ck.lanes == lanes
        if mode == "exact":
            same(one, many)
            same(pk.growth_bound(prob, ctx=c1), pk.growth_bound(prob, ctx=ck))
            assert_bitexact(many, oracle_mm(prob))
        else:
            assert_within(many, oracle_mm(prob), rel=1e-12)
            assert_within(pk.growth_bound(prob, ctx=ck), oracle_mm(prob, "gb"), rel=1e-12)
    finally:
        c1.close()
        ck.close()


@pytest.mark.parametrize("n", [16, 17, 24, 5000])
def test_small_chains_use_at_least_eight_units_per_lane(n):
    """n < 8*lanes: the run uses fewer lanes (each needs >= 8 units so its
    4-unit halo comes from one neighbour); still the oracle's result."""
    prob = chain(n)
    ck = lanes_ctx(3)
    try:
        assert_bitexact(pk.mixed_monotonicity(prob, ctx=ck), oracle_mm(prob))
    finally:
        ck.close()


@pytest.mark.parametrize("g,lanes", [(24, 3), (64, 4), (130, 3)])
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_heat_zslab_lanes(g, lanes, mode):
    prob = heat(g)
    c1, ck = lanes_ctx(1, mode), lanes_ctx(lanes, mode)
    try:
        same(pk.mixed_monotonicity(prob, ctx=c1), pk.mixed_monotonicity(prob, ctx=ck))
        same(pk.growth_bound(prob, ctx=c1), pk.growth_bound(prob, ctx=ck))
    finally:
        c1.close()
        ck.close()


def test_heat_lanes_tiny_remainder_step():
    """Fast mode with a remainder step whose z = hk*kk is below the strip
    kernel's S-form range: that step runs the Horner-in-L 2x2 kernel, in its
    peer-store (Mirror) instantiation on 3 lanes; still bit-identical to one
    lane and within tolerance of the oracle."""
    g = 130
    m = pk.make_heat3d(g)
    n = g ** 3
    rng = np.random.default_rng(41)
    lo = rng.uniform(0.5, 1.0, n)
    hi = lo + rng.uniform(0.0, 0.5, n)
    h = 0.2 / (g - 1) ** 2
    prob = pk.ReachProblem(m, pk.IntervalVector(lo, hi), None, 0.0, 3 * h + 1e-7 * h, h, 1)
    c1, ck = lanes_ctx(1, "fast"), lanes_ctx(3, "fast")
    try:
        a = pk.mixed_monotonicity(prob, ctx=c1)
        same(a, pk.mixed_monotonicity(prob, ctx=ck))
        assert_within(a, oracle_mm(prob))
    finally:
        c1.close()
        ck.close()


def test_workers_argument_maps_to_lanes():
    """The reference's `workers` (reach.hpp:53) selects the lane count: the
    package's process-wide worker contexts, bit-identical results."""
    prob = chain(20000)
    a = pk.mixed_monotonicity(prob, 1)
    b = pk.mixed_monotonicity(prob, 4)
    same(a, b)
    assert b.report.workers == 4
    assert pk.get_worker_context(4).lanes == 4


def test_lane_errors_match_single_lane():
    """Failure keys carry global components: a non-finite value, a box check
    failure and the MM order check report what one lane reports."""
    m = pk.make_traffic(4000)
    bad = pk.ReachProblem(m, pk.IntervalVector(np.full(4000, 1e300), np.full(4000, 1e300)),
                          pk.IntervalVector([4.0], [6.0]), 0.0, 1e6, 1e5, 0)
    c1, ck = lanes_ctx(1), lanes_ctx(3)
    try:
        msgs = []
        for c in (c1, ck):
            with pytest.raises(RuntimeError) as ei:
                pk.mixed_monotonicity(bad, ctx=c)
            msgs.append(str(ei.value))
        assert msgs[0] == msgs[1]
        lo = np.full(4000, 10.0)
        hi = np.full(4000, 20.0)
        lo[3001] = 25.0
        box = pk.ReachProblem(m, pk.IntervalVector(lo, hi, validate=False), pk.IntervalVector([4.0], [6.0]),
                              0.0, 1.0, 0.5, 0)
        with pytest.raises(ValueError, match="lower > upper at component 3001"):
            pk.mixed_monotonicity(box, ctx=ck)
    finally:
        c1.close()
        ck.close()


# ---------------------------------------------------------------- Monte Carlo

@pytest.mark.parametrize("lanes", [2, 3, 7])
def test_mc_lanes_fold_exactly(lanes):
    m = pk.make_laub_loomis()
    c = np.array([1.2, 1.05, 1.5, 2.4, 1.0, 0.1, 0.45])
    prob = pk.ReachProblem(m, pk.IntervalVector(c - 0.05, c + 0.05), None, 0.0, 1.0, 0.005, 20)
    spec = pk.MonteCarloSpec(seed=1, samples_override=20011)
    c1, ck = lanes_ctx(1), lanes_ctx(lanes)
    try:
        one = pk.monte_carlo(prob, spec, ctx=c1)
        many = pk.monte_carlo(prob, spec, ctx=ck)
        same(one, many)
        assert many.report.m == 20011
    finally:
        c1.close()
        ck.close()


def test_mc_fewer_samples_than_lanes():
    """m < workers (reach.cpp:260-264): lanes beyond m get no samples."""
    m, n = pk.make_traffic(6), 6
    prob = pk.ReachProblem(m, pk.IntervalVector(np.full(n, 10.0), np.full(n, 20.0)),
                           pk.IntervalVector([4.0], [6.0]), 0.0, 3.0, 0.5, 2)
    ck = lanes_ctx(8)
    try:
        tube = pk.monte_carlo(prob, pk.MonteCarloSpec(seed=42, samples_override=3), ctx=ck)
        ref = O.monte_carlo(m, np.full(n, 10.0), np.full(n, 20.0), [4.0], [6.0], 0.0, 3.0, 0.5, 2, 42, 3)
        assert_bitexact(tube, ref)
    finally:
        ck.close()


def test_mc_range_pieces_fold_to_the_whole():
    """pirk_monte_carlo_range (the per-rank piece of a sample-sharded run)
    over 3 uneven ranges, folded, equals one monte_carlo call bit for bit."""
    m = pk.make_arch_quadrotor()
    lo = np.array([-0.4] * 6 + [0.0] * 6)
    prob = pk.ReachProblem(m, pk.IntervalVector(lo, -lo), None, 0.0, 0.5, 0.01, 10)
    total = 9001
    ctx = lanes_ctx(1)
    try:
        whole = pk.monte_carlo(prob, pk.MonteCarloSpec(seed=5, samples_override=total), ctx=ctx)
        S = len(whole.entries)
        flo = np.full((S, 12), np.inf)
        fhi = np.full((S, 12), -np.inf)
        for b, e in ((0, 1234), (1234, 1235), (1235, total)):
            pk.monte_carlo_range(prob, 5, b, e, flo, fhi, ctx=ctx)
        _, wl, wh = tube_arrays(whole)
        assert np.array_equal(flo, wl) and np.array_equal(fhi, wh)
        # and the oracle's ranges agree
        ref = O.monte_carlo(m, lo, -lo, None, None, 0.0, 0.5, 0.01, 10, 5, total, 1234, 1235)
        a = np.full((S, 12), np.inf)
        b_ = np.full((S, 12), -np.inf)
        pk.monte_carlo_range(prob, 5, 1234, 1235, a, b_, ctx=ctx)
        assert np.allclose(a, ref.lower, rtol=1e-12, atol=1e-14)
    finally:
        ctx.close()


def test_release_cache_frees_state():
    import torch

    prob = traffic(2_000_000, stride=0, t1=1.0)
    ctx = lanes_ctx(1)
    try:
        pk.mixed_monotonicity(prob, ctx=ctx)
        free0, _ = torch.cuda.mem_get_info()
        ctx.release_cache()
        free1, _ = torch.cuda.mem_get_info()
        assert free1 - free0 >= 4 * 2_000_000 * 8 * 0.9
    finally:
        ctx.close()


def test_copy_engine_halo_path():
    """PIRK_LANE_HALO=copy: halos by cudaMemcpyPeerAsync on the copy stream
    instead of the fused peer stores of the boundary launches (the fallback
    for lanes without peer access) -- same bit-identical results.  The env
    var is read once per process, so the lane tests rerun in a child."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PIRK_LANE_HALO="copy")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(root, "tests", "test_gpu_multilane.py"), "-k", "lanes and not copy and not split"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_split_lane_schedule():
    """PIRK_LANE_SCHEDULE=split: boundary units as separate launches first
    (their peer stores overlap the interior launch) instead of the default one
    launch per lane and step -- same bit-identical results."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PIRK_LANE_SCHEDULE="split")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(root, "tests", "test_gpu_multilane.py"), "-k", "lanes and not copy and not split"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
