"""GPU parity: the CUDA path (through the C ABI) against the oracle on
identical inputs.  Exact mode must be bit-identical; fast mode within the
SURVEY.md 8(d) tolerance contract (relative <= 1e-12, never tighter)."""
import numpy as np
import pytest

import paper_2001_10635_b200 as pk
from oracle import oracle as O
from tests.helpers import assert_bitexact, assert_within, tube_arrays

pytestmark = pytest.mark.gpu


def traffic_problem(n, t1=30.0, h=0.5, stride=10, lo=10.0, hi=20.0, plo=4.0, phi=6.0):
    m = pk.make_traffic(n)
    return m, pk.ReachProblem(m, pk.IntervalVector(np.full(n, lo), np.full(n, hi)),
                              pk.IntervalVector([plo], [phi]), 0.0, t1, h, stride)


def heat_problem(g, t1=0.05, h=0.002, stride=5, lo=None, hi=None):
    m = pk.make_heat3d(g)
    n = g ** 3
    lo = np.full(n, 0.9) if lo is None else lo
    hi = np.full(n, 1.1) if hi is None else hi
    return m, pk.ReachProblem(m, pk.IntervalVector(lo, hi), None, 0.0, t1, h, stride)


def chain_problem(n, t1=1.0, h=0.01, stride=10):
    m = pk.make_chain(n)
    c = 2.0 * np.array([O.u01(7, 0, i) for i in range(n)]) - 1.0
    return m, pk.ReachProblem(m, pk.IntervalVector(c - 0.05, c + 0.05),
                              pk.IntervalVector([-0.1], [0.1]), 0.0, t1, h, stride)


def oracle_for(method, prob):
    p = prob
    plo = p.inputs.lower if p.inputs is not None else None
    phi = p.inputs.upper if p.inputs is not None else None
    fn = {"mm": O.mixed_monotonicity, "gb": O.growth_bound}[method]
    return fn(p.model, p.initial.lower, p.initial.upper, plo, phi, p.t0, p.t1, p.h, p.tube_stride)


# ------------------------------------------------------------------ traffic

@pytest.mark.parametrize("n", [3, 5, 50, 1000, 1017, 2033, 100003])
def test_traffic_mm_exact(ctx, n):
    m, prob = traffic_problem(n)
    assert_bitexact(pk.mixed_monotonicity(prob, ctx=ctx), oracle_for("mm", prob))


@pytest.mark.parametrize("n", [3, 5, 1000, 5001])
def test_traffic_gb_exact(ctx, n):
    m, prob = traffic_problem(n)
    assert_bitexact(pk.growth_bound(prob, ctx=ctx), oracle_for("gb", prob))


def test_traffic_ragged_box_and_remainder_step(ctx):
    # non-uniform box, h that does not divide the span (shortened last step,
    # rk4.cpp:100) and a stride that does not divide the step count
    n = 777
    rng = np.random.default_rng(3)
    lo = rng.uniform(0, 300, n)
    hi = lo + rng.uniform(0, 20, n)
    m = pk.make_traffic(n)
    prob = pk.ReachProblem(m, pk.IntervalVector(lo, hi), pk.IntervalVector([0.5], [30.0]),
                           0.0, 10.0, 0.3, 7)
    assert_bitexact(pk.mixed_monotonicity(prob, ctx=ctx), oracle_for("mm", prob))
    assert_bitexact(pk.growth_bound(prob, ctx=ctx), oracle_for("gb", prob))


def test_traffic_fast_mode_tolerance(fast_ctx):
    m, prob = traffic_problem(5000)
    assert_within(pk.mixed_monotonicity(prob, ctx=fast_ctx), oracle_for("mm", prob))
    assert_within(pk.growth_bound(prob, ctx=fast_ctx), oracle_for("gb", prob))


# --------------------------------------------------------------------- heat

@pytest.mark.parametrize("g", [2, 3, 4, 5, 8, 31, 33, 40])
def test_heat_mm_exact(ctx, g):
    m, prob = heat_problem(g, t1=0.02, h=0.2 / (g - 1) ** 2 if g > 3 else 0.002, stride=3)
    assert_bitexact(pk.mixed_monotonicity(prob, ctx=ctx), oracle_for("mm", prob))


def test_heat_ragged_box(ctx):
    g = 20
    n = g ** 3
    rng = np.random.default_rng(11)
    lo = rng.uniform(0.5, 1.0, n)
    hi = lo + rng.uniform(0.0, 0.5, n)
    m, prob = heat_problem(g, t1=0.005, h=0.0004, stride=4, lo=lo, hi=hi)
    assert_bitexact(pk.mixed_monotonicity(prob, ctx=ctx), oracle_for("mm", prob))
    assert_bitexact(pk.growth_bound(prob, ctx=ctx), oracle_for("gb", prob))


@pytest.mark.parametrize("g", [8, 37])
def test_heat_fast_mode_tolerance(fast_ctx, g):
    m, prob = heat_problem(g, t1=0.2 / (g - 1) ** 2 * 20, h=0.2 / (g - 1) ** 2, stride=5)
    assert_within(pk.mixed_monotonicity(prob, ctx=fast_ctx), oracle_for("mm", prob))


def heat_interior_problem(g, seed=5, steps=4):
    """A grid large enough for interior tiles (halo-4 footprint inside the
    grid: g >= 68), the path the bench sizes run; g = 160 also splits z into
    chunks, odd g takes the cp.async fallback instead of TMA."""
    n = g ** 3
    rng = np.random.default_rng(seed)
    lo = rng.uniform(0.5, 1.0, n)
    hi = lo + rng.uniform(0.0, 0.5, n)
    h = 0.2 / (g - 1) ** 2
    return heat_problem(g, t1=steps * h, h=h, stride=2, lo=lo, hi=hi)


@pytest.mark.parametrize("g", [72, 75, 100, 160])
def test_heat_interior_tiles_exact(ctx, g):
    m, prob = heat_interior_problem(g)
    assert_bitexact(pk.mixed_monotonicity(prob, ctx=ctx), oracle_for("mm", prob))
    if g == 100:
        assert_bitexact(pk.growth_bound(prob, ctx=ctx), oracle_for("gb", prob))


@pytest.mark.parametrize("g", [72, 75, 160])
def test_heat_interior_tiles_fast(fast_ctx, g):
    m, prob = heat_interior_problem(g)
    assert_within(pk.mixed_monotonicity(prob, ctx=fast_ctx), oracle_for("mm", prob))


def test_heat_fast_mode_long_run(fast_ctx):
    """100 fast-mode steps on interior tiles: the restructured arithmetic
    (Horner form of RK4 for the linear field, shared partial sums) stays
    within the 1e-12 contract over a full-length reach."""
    m, prob = heat_interior_problem(72, seed=9, steps=100)
    assert_within(pk.mixed_monotonicity(prob, ctx=fast_ctx), oracle_for("mm", prob))
    assert_within(pk.growth_bound(prob, ctx=fast_ctx), oracle_for("gb", prob))


@pytest.mark.parametrize("z", [1.0 / 6.0, 0.02, 2e-6])
def test_heat_fast_sform_z_range(fast_ctx, z):
    """The strip kernel evaluates RK4 as a polynomial in the neighbour-sum
    operator S (heat.cuh heat_sform_coeffs); its stage coefficients are
    q3/q4, q2/q4, q1/q4.  z = h*kk = 1/6 is the root of q3 (a Horner form in S
    with q_k/q_{k+1} coefficients would divide by zero there); 2e-6 is near
    the small-z limit of the S form (stage values ~24/z^3 |x|)."""
    g = 72
    n = g ** 3
    rng = np.random.default_rng(21)
    lo = rng.uniform(0.5, 1.0, n)
    hi = lo + rng.uniform(0.0, 0.5, n)
    h = z / (g - 1) ** 2
    m, prob = heat_problem(g, t1=6 * h, h=h, stride=2, lo=lo, hi=hi)
    assert_within(pk.mixed_monotonicity(prob, ctx=fast_ctx), oracle_for("mm", prob))


@pytest.mark.parametrize("g", [72, 162])
def test_heat_fast_tiny_remainder_step(fast_ctx, g):
    """A remainder step with z = hk*kk far below the S form's range runs the
    Horner-in-L kernel for that step (launch_heat_step); g = 162 (n >= 2^22,
    final box only) is the field-pipelined driver's case, which then takes the
    per-step path (engine.cu heat_plan_strip_ok)."""
    n = g ** 3
    rng = np.random.default_rng(23)
    lo = rng.uniform(0.5, 1.0, n)
    hi = lo + rng.uniform(0.0, 0.5, n)
    h = 0.2 / (g - 1) ** 2
    t1 = 3 * h + 1e-7 * h
    stride = 0 if g == 162 else 1
    m, prob = heat_problem(g, t1=t1, h=h, stride=stride, lo=lo, hi=hi)
    ref = oracle_for("mm", prob)
    assert len(ref.times) == (1 if stride == 0 else 5)
    assert_within(pk.mixed_monotonicity(prob, ctx=fast_ctx), ref)


@pytest.mark.parametrize("variant", ["1x2", "2x2", "strip"])
def test_heat_block_variants(variant):
    """Both heat kernels (1x2 pairs, 2x2 blocks) in both modes: the selector
    (PIRK_HEAT_BLOCK) is read once per process, so each runs in a child."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PIRK_HEAT_BLOCK=variant)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(root, "tests", "test_gpu_parity.py"),
                        "-k", "heat and not variants"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("variant", ["warp", "warp_single_step"])
def test_chain_kernel_variants(variant):
    """The chain kernels in both modes on the traffic and coupled-chain tests:
    shared-memory tiles, the warp-tiled kernel (default: two RK4 steps per
    launch in full-domain runs) and the warp-tiled kernel one step at a time."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PIRK_CHAIN_KERNEL=variant.split("_")[0])
    if variant == "warp_single_step":
        env["PIRK_CHAIN_FUSE"] = "0"
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(root, "tests", "test_gpu_parity.py"),
                        "-k", "(traffic or chain) and not variant"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


# -------------------------------------------------------------------- chain

@pytest.mark.parametrize("n", [1, 2, 7, 1000, 1016, 1017, 5000])
def test_chain_mm_exact(ctx, n):
    m, prob = chain_problem(n)
    assert_bitexact(pk.mixed_monotonicity(prob, ctx=ctx), oracle_for("mm", prob))


def test_chain_fast_mode_tolerance(fast_ctx):
    m, prob = chain_problem(3000)
    assert_within(pk.mixed_monotonicity(prob, ctx=fast_ctx), oracle_for("mm", prob), atol=1e-15)


# ------------------------------------------------------------ small systems

def test_scalar_linear_mm_is_e_2e(ctx):
    # test_reach.cpp:70-75 / acceptance criterion 5
    m = pk.make_scalar_linear()
    prob = pk.ReachProblem(m, pk.IntervalVector([1.0], [2.0]), None, 0.0, 1.0, 0.001, 0)
    tube = pk.mixed_monotonicity(prob, ctx=ctx)
    fin = tube.entries[-1].box
    assert abs(fin.lower[0] - np.e) <= 1e-4 and abs(fin.upper[0] - 2 * np.e) <= 1e-4
    assert_bitexact(tube, oracle_for("mm", prob))


def test_frozen_system_keeps_box(ctx):
    # test_reach.cpp:35-50
    m = pk.make_zero(2)
    init = pk.IntervalVector([0.0, 0.0], [1.0, 1.0])
    prob = pk.ReachProblem(m, init, None, 0.0, 1.0, 0.1, 4)
    for tube in (pk.growth_bound(prob, ctx=ctx), pk.mixed_monotonicity(prob, ctx=ctx)):
        assert len(tube.entries) >= 2
        for e in tube.entries:
            assert e.box == init
        assert tube.entries[-1].t == 1.0
    mc = pk.monte_carlo(pk.ReachProblem(m, init, None, 0.0, 1.0, 0.1, 0),
                        pk.MonteCarloSpec(samples_override=100), ctx=ctx)
    assert pk.subset_of(mc.entries[-1].box, init)


def test_scalar_decay_gb_closed_form(ctx):
    # test_reach.cpp:53-68 / acceptance criterion 4
    m = pk.make_scalar_decay()
    prob = pk.ReachProblem(m, pk.IntervalVector([0.9], [1.1]), pk.IntervalVector([0.0], [0.0]),
                           0.0, 1.0, 0.001, 0)
    tube = pk.growth_bound(prob, ctx=ctx)
    fin = tube.entries[-1].box
    assert abs((fin.upper[0] - fin.lower[0]) / 2 - 0.1 / np.e) <= 1e-5
    assert tube.report.steps == 1000
    assert_bitexact(tube, oracle_for("gb", prob))


def test_laub_loomis_gb_exact(ctx):
    m = pk.make_laub_loomis()
    lo = np.array([1.15, 1.00, 1.45, 2.35, 0.95, 0.05, 0.40])
    prob = pk.ReachProblem(m, pk.IntervalVector(lo, lo + 0.1), None, 0.0, 1.0, 0.005, 20)
    assert_bitexact(pk.growth_bound(prob, ctx=ctx), oracle_for("gb", prob))


def test_laub_loomis_jacobian_mm_exact(ctx):
    m = pk.with_jacobian_decomposition(pk.make_laub_loomis())
    lo = np.array([1.15, 1.00, 1.45, 2.35, 0.95, 0.05, 0.40])
    prob = pk.ReachProblem(m, pk.IntervalVector(lo, lo + 0.1), None, 0.0, 0.2, 0.005, 10)
    assert_bitexact(pk.mixed_monotonicity(prob, ctx=ctx), oracle_for("mm", prob))


def arch_quad_problem(stride=10, decomp=False):
    m = pk.make_arch_quadrotor()
    if decomp:
        m = pk.with_jacobian_decomposition(m)
    lo = np.array([-0.4] * 6 + [0.0] * 6)
    return m, pk.ReachProblem(m, pk.IntervalVector(lo, -lo), None, 0.0, 1.0, 0.01, stride)


def test_arch_quad_gb_tolerance(ctx):
    # config 1 as shipped (growth bound); CUDA sin/cos vs glibc -> tolerance
    m, prob = arch_quad_problem()
    assert_within(pk.growth_bound(prob, ctx=ctx), oracle_for("gb", prob), rel=1e-12, atol=1e-14)


def test_arch_quad_ctmm_tolerance(ctx):
    # config 1 as CTMM through the Jacobian-bound decomposition
    m, prob = arch_quad_problem(decomp=True)
    assert_within(pk.mixed_monotonicity(prob, ctx=ctx), oracle_for("mm", prob), rel=1e-12,
                  atol=1e-14)


# -------------------------------------------------------------- Monte Carlo

def mc_oracle(prob, seed, m):
    p = prob
    plo = p.inputs.lower if p.inputs is not None else None
    phi = p.inputs.upper if p.inputs is not None else None
    return O.monte_carlo(p.model, p.initial.lower, p.initial.upper, plo, phi, p.t0, p.t1, p.h,
                         p.tube_stride, seed, m)


def test_laub_loomis_mc_exact(ctx):
    m = pk.make_laub_loomis()
    c = np.array([1.2, 1.05, 1.5, 2.4, 1.0, 0.1, 0.45])
    prob = pk.ReachProblem(m, pk.IntervalVector(c - 0.05, c + 0.05), None, 0.0, 1.0, 0.005, 20)
    tube = pk.monte_carlo(prob, pk.MonteCarloSpec(seed=1, samples_override=3000), ctx=ctx)
    assert_bitexact(tube, mc_oracle(prob, 1, 3000))
    assert tube.report.m == 3000


def test_traffic_mc_exact_and_seeded(ctx):
    # test_reach.cpp:88-111: traffic n=6, seed 42, m=64, stride 2
    m, prob = traffic_problem(6, t1=3.0, h=0.5, stride=2)
    a = pk.monte_carlo(prob, pk.MonteCarloSpec(seed=42, samples_override=64), ctx=ctx)
    assert_bitexact(a, mc_oracle(prob, 42, 64))
    b = pk.monte_carlo(prob, pk.MonteCarloSpec(seed=43, samples_override=64), ctx=ctx)
    assert pk.tube_to_csv(a) != pk.tube_to_csv(b)
    c3 = pk.monte_carlo(prob, pk.MonteCarloSpec(seed=42, samples_override=3), ctx=ctx)
    assert_bitexact(c3, mc_oracle(prob, 42, 3))


def test_arch_quad_mc_tolerance(ctx):
    m, prob = arch_quad_problem()
    tube = pk.monte_carlo(prob, pk.MonteCarloSpec(seed=1, samples_override=4096), ctx=ctx)
    assert_within(tube, mc_oracle(prob, 1, 4096), rel=1e-12, atol=1e-14)


def test_arch_quad_mc_fast_mode_tolerance(fast_ctx):
    """Fast mode: small-angle sincos and folded quotients in the arch-quadrotor
    field (csrc/small.cuh aq_f_all_fast), against the glibc-trig oracle."""
    m, prob = arch_quad_problem()
    tube = pk.monte_carlo(prob, pk.MonteCarloSpec(seed=1, samples_override=4096), ctx=fast_ctx)
    assert_within(tube, mc_oracle(prob, 1, 4096), rel=1e-12, atol=1e-14)


def test_mc_hull_inside_exact_image(ctx):
    # test_reach.cpp:113-124
    m = pk.make_scalar_linear()
    prob = pk.ReachProblem(m, pk.IntervalVector([1.0], [2.0]), None, 0.0, 1.0, 0.001, 0)
    fin = pk.monte_carlo(prob, pk.MonteCarloSpec(seed=3, samples_override=1000), ctx=ctx).entries[-1].box
    e = np.e
    assert fin.lower[0] >= e - 1e-9 and fin.upper[0] <= 2 * e + 1e-9
    assert fin.lower[0] <= e * 1.02 and fin.upper[0] >= 2 * e * 0.98


def test_coverage_estimate_matches_oracle(ctx):
    # test_reach.cpp:126-147
    m = pk.make_zero(2)
    prob = pk.ReachProblem(m, pk.IntervalVector([0.0, 0.0], [1.0, 1.0]), None, 0.0, 1.0, 0.1, 0)
    spec = pk.MonteCarloSpec(seed=5, samples_override=200)
    tube = pk.monte_carlo(prob, spec, ctx=ctx)
    honest = pk.coverage_estimate(prob, spec, tube, 5000, 77, ctx=ctx)
    fin = tube.entries[-1].box
    ref = O.coverage_estimate(m, [0, 0], [1, 1], None, None, 0.0, 1.0, 0.1, fin.lower, fin.upper,
                              5000, 77)
    assert honest == ref
    assert 0.0 <= honest < 0.2


# ------------------------------------------------------------------- errors

def test_non_finite_reports_step(ctx):
    # test_rk4.cpp:138-154 through mixed monotonicity
    m = pk.make_scalar_linear(5.0)
    prob = pk.ReachProblem(m, pk.IntervalVector([1.0], [1.0]), None, 0.0, 600.0, 10.0, 0)
    with pytest.raises(RuntimeError) as ei:
        pk.mixed_monotonicity(prob, ctx=ctx)
    with pytest.raises(O.OracleError) as eo:
        oracle_for("mm", prob)
    assert str(ei.value) == str(eo.value)


def test_non_finite_large_model(ctx):
    # traffic driven to overflow by an absurd step: error names step/component
    m, prob = traffic_problem(2000, t1=1e6, h=1e5, stride=0, lo=1e300, hi=1e300)
    with pytest.raises(RuntimeError) as ei:
        pk.mixed_monotonicity(prob, ctx=ctx)
    with pytest.raises(O.OracleError) as eo:
        oracle_for("mm", prob)
    assert str(ei.value) == str(eo.value)


def test_order_violation_reported(ctx):
    # test_reach.cpp:190-206 uses a custom decomposition; the chain model with
    # an inverted box is the closest catalog analogue: check the message
    # matches the oracle's exactly.
    m = pk.make_chain(50, a=-3.0, b=2.0, c=-2.0)
    c = np.linspace(-1, 1, 50)
    prob = pk.ReachProblem(m, pk.IntervalVector(c - 0.5, c + 0.5), pk.IntervalVector([-1.0], [1.0]),
                           0.0, 3.0, 0.1, 1)
    try:
        ref = oracle_for("mm", prob)
    except O.OracleError as e:
        with pytest.raises(RuntimeError) as ei:
            pk.mixed_monotonicity(prob, ctx=ctx)
        assert str(ei.value) == str(e)
    else:
        assert_bitexact(pk.mixed_monotonicity(prob, ctx=ctx), ref)


def test_unsupported_model_is_loud(ctx):
    m = pk.make_traffic(2000)  # Monte Carlo kernels hold a sample in registers: n <= 1024
    prob = pk.ReachProblem(m, pk.IntervalVector(np.zeros(2000), np.ones(2000)),
                           pk.IntervalVector([1.0], [2.0]), 0.0, 1.0, 0.5, 0)
    with pytest.raises(NotImplementedError):
        pk.monte_carlo(prob, pk.MonteCarloSpec(samples_override=10), ctx=ctx)


def test_missing_capabilities_rejected(ctx):
    m = pk.make_chain(10)
    prob = pk.ReachProblem(m, pk.IntervalVector(np.zeros(10), np.ones(10)),
                           pk.IntervalVector([0.0], [0.0]), 0.0, 1.0, 0.1, 0)
    with pytest.raises(ValueError, match="no deviation dynamics"):
        pk.growth_bound(prob, ctx=ctx)
    ll = pk.make_laub_loomis()
    prob2 = pk.ReachProblem(ll, pk.IntervalVector(np.zeros(7), np.ones(7)), None, 0.0, 1.0, 0.1, 0)
    with pytest.raises(ValueError, match="no decomposition"):
        pk.mixed_monotonicity(prob2, ctx=ctx)


# ------------------------------------------- golden vectors from the reference

GOLDEN = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "golden.npz")


def _golden_cases():
    from tests.golden.make_golden import cases
    return cases()


@pytest.mark.parametrize("case", _golden_cases(), ids=lambda c: c[0])
def test_cuda_matches_reference_golden(ctx, case):
    """The CUDA path against vectors produced by the reference itself."""
    name, method, model, lo, hi, plo, phi, t0, t1, h, stride, kw = case
    g = np.load(GOLDEN)

    class R:
        times = g[f"{name}__times"]
        lower = g[f"{name}__lower"]
        upper = g[f"{name}__upper"]

    n = model.dim
    init = pk.IntervalVector(np.broadcast_to(np.asarray(lo, float), (n,)),
                             np.broadcast_to(np.asarray(hi, float), (n,)))
    inputs = pk.IntervalVector(plo, phi) if plo is not None else None
    prob = pk.ReachProblem(model, init, inputs, t0, t1, h, stride)
    if method == O.METHOD_MM:
        tube = pk.mixed_monotonicity(prob, ctx=ctx)
    elif method == O.METHOD_GB:
        tube = pk.growth_bound(prob, ctx=ctx)
    else:
        tube = pk.monte_carlo(prob, pk.MonteCarloSpec(seed=kw["seed"], samples_override=kw["samples"]),
                              ctx=ctx)
    if model.kind == pk.ARCH_QUAD:  # CUDA sin/cos vs glibc: tolerance contract
        assert_within(tube, R, rel=1e-12, atol=1e-14)
    else:
        assert_bitexact(tube, R)


# ------------------------------------------------------------ formats / driver

def test_tube_formats_match_reference_io(ctx):
    """The CUDA tube of traffic n=5 through tube_to_csv / tube_to_json is
    byte-identical to the reference's io.cpp output (tests/golden/io, written by
    oracle/ref_io_golden.cpp); only the report's wall-clock phases differ and
    are taken from the golden file."""
    import json
    import os
    from paper_2001_10635_b200 import driver as D
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")
    m = pk.make_traffic(5)
    prob = pk.ReachProblem(m, pk.IntervalVector(np.full(5, 10.0), np.full(5, 20.0)),
                           pk.IntervalVector([4.0], [6.0]), 0.0, 3.0, 0.5, 2)
    tube = D.dispatch("mixed-monotonicity", prob, ctx=ctx)
    with open(os.path.join(gold, "traffic_mm.csv")) as f:
        assert D.tube_to_csv(tube) == f.read()
    with open(os.path.join(gold, "traffic_mm.json")) as f:
        text = f.read()
    ref_rep = json.loads(text)["report"]
    for k in ("method", "n", "m", "workers", "steps", "peak_state_bytes"):
        assert getattr(tube.report, k) == ref_rep[k], k
    ph = ref_rep["phases"]
    tube.report.phases = pk.PhaseTimes(ph["setup_s"], ph["integration_s"], ph["reduction_s"])
    assert D.tube_to_json(tube) == text


def test_driver_bench_sweep_on_device(ctx):
    """driver.bench over two traffic sizes and the CSV the reference's bench
    command prints."""
    from paper_2001_10635_b200 import driver as D
    rows = D.bench("traffic", "mixed-monotonicity", [100, 1000], [1], 2, 0.0, 3.0, 0.5, ctx=ctx)
    assert [(r.n, r.status, r.steps) for r in rows] == [(100, "ok", 6), (1000, "ok", 6)]
    lines = D.bench_csv(rows).splitlines()
    assert lines[0] == "n,workers,median_seconds,steps,status" and len(lines) == 3


# ------------------------------------------------------------ sharded windows

class _NoopExchanger:
    """Halo exchange stand-in for virtual ranks on one device: the test copies
    the halos before each exchange step, so start/finish only mark the split
    (interior launch, then boundary launches) that ShardedReach.run makes."""

    def start(self, fields):
        return None

    def finish(self, handle):
        pass

    def exchange(self, fields):
        pass


def _fill_halos(runs, unit):
    """Copy every rank's owned boundary units into its neighbours' halos."""
    for r, run in enumerate(runs):
        s = run.shard
        for nb in (r - 1, r + 1):
            if nb < 0 or nb >= len(runs):
                continue
            o = runs[nb].shard
            lo, hi = (s.win_begin, s.begin) if nb == r - 1 else (s.end, s.win_end)
            for f in (0, 1):
                src = runs[nb].a[f][(lo - o.win_begin) * unit:(hi - o.win_begin) * unit]
                run.a[f][(lo - s.win_begin) * unit:(hi - s.win_begin) * unit].copy_(src)


@pytest.mark.parametrize("kind,world,K,mode", [("heat", 3, 1, "fast"), ("heat", 3, 2, "exact"),
                                               ("heat", 2, 1, "exact"), ("traffic", 3, 2, "fast"),
                                               ("chain", 2, 1, "exact")])
def test_sharded_windows_on_device(kind, world, K, mode):
    """The N>1 data path on one B200: virtual ranks run ShardedReach with the
    CUDA windowed step (interior launch + boundary launches on exchange steps,
    deep halos for K > 1) and reproduce the single-device reach bit for bit --
    the windowed heat strip / chain warp kernels compute each unit exactly as
    the full-domain launch does."""
    import torch
    from paper_2001_10635_b200 import sharded as S
    c = pk.Context(0, mode)
    try:
        if kind == "heat":
            g = 64
            m = pk.make_heat3d(g)
            n = m.dim
            lo = 0.9 - 0.05 * ((np.arange(n) * 7) % 5)
            hi = lo + 0.2
            plo = phi = None
            h = 0.2 / (g - 1) ** 2
            t1 = 6 * h
        else:
            n = 5000
            m = pk.make_traffic(n) if kind == "traffic" else pk.make_chain(n)
            lo = (10.0 if kind == "traffic" else -0.05) + 0.001 * (np.arange(n) % 7)
            hi = lo + (10.0 if kind == "traffic" else 0.1)
            plo, phi = ([4.0], [6.0]) if kind == "traffic" else ([-0.1], [0.1])
            h, t1 = (0.5, 3.0) if kind == "traffic" else (0.01, 0.06)
        prob = pk.ReachProblem(m, pk.IntervalVector(lo, hi), pk.IntervalVector(plo, phi) if plo else None,
                               0.0, t1, h, 0)
        ref = pk.mixed_monotonicity(prob, ctx=c).entries[-1].box
        units, unit = S.units_of(m)
        step = S.device_step_fn(m, "mixed-monotonicity", c)
        runs = []
        for r in range(world):
            sh = S.Shard(units, world, r, 4 * K)
            run = S.ShardedReach(m, "mixed-monotonicity", sh, step, _NoopExchanger(), plo, phi, K=K)
            run.alloc(lambda k: torch.full((k,), float("nan"), dtype=torch.float64, device="cuda"))
            sl = slice(sh.win_begin * unit, sh.win_end * unit)
            run.a[0].copy_(torch.from_numpy(np.ascontiguousarray(lo[sl])))
            run.a[1].copy_(torch.from_numpy(np.ascontiguousarray(hi[sl])))
            runs.append(run)
        for i, (t, hk) in enumerate(S.plan_rk4_steps(0.0, t1, h)):
            if i % K == 0:
                _fill_halos(runs, unit)
            for run in runs:
                run.run([(t, hk)], i)
        torch.cuda.synchronize()
        got_lo, got_hi = np.empty(n), np.empty(n)
        for run in runs:
            o0, o1 = run.owned()
            b, e = run.shard.begin * unit, run.shard.end * unit
            got_lo[b:e], got_hi[b:e] = o0.cpu().numpy(), o1.cpu().numpy()
        assert np.array_equal(got_lo, ref.lower) and np.array_equal(got_hi, ref.upper)
    finally:
        c.close()


# ------------------------------------------------------------ field-pipelined heat CTMM

@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_heat_pipelined_final_box(mode):
    """heat3d CTMM with only the final box and n >= 2^22 takes the field-
    pipelined driver (engine.cu run_heat_mm_pipelined: lower field integrated
    while the upper field uploads, lower field downloaded while the upper one
    integrates).  Same result as the oracle: bit-exact / within tolerance."""
    g = 170  # n = 4.913e6
    n = g ** 3
    rng = np.random.default_rng(11)
    lo = rng.uniform(0.5, 1.0, n)
    hi = lo + rng.uniform(0.0, 0.5, n)
    h = 0.2 / (g - 1) ** 2
    m, prob = heat_problem(g, t1=3 * h, h=h, stride=0, lo=lo, hi=hi)
    c = pk.Context(0, mode)
    try:
        tube = pk.mixed_monotonicity(prob, ctx=c)
        ref = oracle_for("mm", prob)
        if mode == "exact":
            assert_bitexact(tube, ref)
        else:
            assert_within(tube, ref)
        bad = lo.copy()
        bad[12345] = hi[12345] + 1.0
        prob2 = pk.ReachProblem(m, pk.IntervalVector(bad, hi, validate=False), None, 0.0, 3 * h, h, 0)
        with pytest.raises(ValueError, match="lower > upper at component 12345"):
            pk.mixed_monotonicity(prob2, ctx=c)
    finally:
        c.close()


_SKEW_CHILD = r"""
import sys, numpy as np, paper_2001_10635_b200 as pk
g, steps, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
n = g ** 3
rng = np.random.default_rng(5)
lo = rng.uniform(0.5, 1.0, n)
hi = lo + rng.uniform(0.0, 0.5, n)
h = 0.2 / (g - 1) ** 2
m = pk.make_heat3d(g)
prob = pk.ReachProblem(m, pk.IntervalVector(lo, hi), None, 0.0, steps * h, h, 0)
c = pk.Context(0, "fast")
t = pk.mixed_monotonicity(prob, ctx=c)
np.save(out + "_lo.npy", t.entries[-1].box.lower); np.save(out + "_hi.npy", t.entries[-1].box.upper)
"""


def test_heat_pipelined_skew_schedules_identical(tmp_path):
    """The field-pipelined driver's skewed rounds (engine.cu skew_fronts:
    strips of S planes, lower field started before its upload completes,
    upper field downloaded S planes at a time) give bit-identical boxes for any
    strip width, including the unskewed schedule (PIRK_SKEW=0) and strips
    narrower than the 4-plane step cone, and stay within the fast-mode
    tolerance of the oracle."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    g, steps = 162, 24  # n = 4.25e6 >= 2^22; 24 steps: the step cone spans 92 planes
    res = {}
    for name, env in (("noskew", {"PIRK_SKEW": "0"}), ("s8", {"PIRK_SKEW_S": "8"}),
                      ("s3", {"PIRK_SKEW_S": "3", "PIRK_SKEW_S0": "5", "PIRK_SKEW_J": "7"}),
                      ("s40", {"PIRK_SKEW_S": "40", "PIRK_SKEW_J": "1"}), ("default", {})):
        out = str(tmp_path / name)
        r = subprocess.run([sys.executable, "-c", _SKEW_CHILD, str(g), str(steps), out],
                           env=dict(os.environ, **env), cwd=root, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        res[name] = (np.load(out + "_lo.npy"), np.load(out + "_hi.npy"))
    for name in res:
        assert np.array_equal(res[name][0], res["noskew"][0]), name
        assert np.array_equal(res[name][1], res["noskew"][1]), name
    n = g ** 3
    rng = np.random.default_rng(5)
    lo = rng.uniform(0.5, 1.0, n)
    hi = lo + rng.uniform(0.0, 0.5, n)
    h = 0.2 / (g - 1) ** 2
    m, prob = heat_problem(g, t1=steps * h, h=h, stride=0, lo=lo, hi=hi)
    ref = oracle_for("mm", prob)
    for f, r in ((0, ref.lower[-1]), (1, ref.upper[-1])):
        got = res["default"][f]
        assert np.max(np.abs(got - r) / np.abs(r)) <= 1e-12


def test_small_serial_kernel_variant():
    """The one-thread small-system integrator (PIRK_SMALL_SERIAL=1) and the
    default warp-parallel one give the same results: the small-system tests
    rerun in a child process with the serial kernel."""
    import os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PIRK_SMALL_SERIAL="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        os.path.join(root, "tests", "test_gpu_parity.py"),
                        "-k", "scalar or laub or arch_quad_gb or arch_quad_ctmm or frozen or golden"],
                       env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_arch_quad_fast_mode_small_integrator(fast_ctx):
    """Fast mode: the warp-parallel small integrator evaluates the arch-quadrotor
    with the small-angle sincos of the MC kernel -- GB and CTMM within the
    tolerance contract of the glibc-trig oracle."""
    m, prob = arch_quad_problem()
    assert_within(pk.growth_bound(prob, ctx=fast_ctx), oracle_for("gb", prob), rel=1e-12, atol=1e-14)
    m, prob = arch_quad_problem(decomp=True)
    assert_within(pk.mixed_monotonicity(prob, ctx=fast_ctx), oracle_for("mm", prob), rel=1e-12, atol=1e-14)
