"""Parity at the sizes the bench runs (VERDICT r1 "next" #1).

Every case runs the CUDA path through the package API and compares with the
reference itself (oracle/_ref, the unmodified /root/reference/proj/src built by
oracle/Makefile and driven through its own ivreach:: entry points on all host
cores), or -- for C5 at its full n = 4.096e9, which no CPU here can hold -- with
a size-independent exact restatement (oracle.heat_line_uniform: from a uniform
box the heat field is constant on every (y, z) plane, so every one of the 4e9
components must equal a 1-D line computed in reference arithmetic).

Exact mode: bit-identical (== semantics).  Fast mode: relative <= 1e-12
(SURVEY.md 8(d)), tolerance written in each assertion.
"""
import os

import numpy as np
import pytest

import paper_2001_10635_b200 as pk
from oracle import oracle as O
from tests.helpers import assert_bitexact, assert_within

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

# bench.py runs C5 at h = 5e-8 on g = 1600: h * alpha/delta^2 = 5e-8 * 1599^2
BENCH_HKK = 5e-8 * 1599.0 ** 2


def _need_ref():
    if not O.ref_available():
        pytest.fail("oracle/_ref/libivreach_ref.so missing: run __graft_entry__.build() "
                    "where /root/reference is present (the .so travels with the snapshot)")
    return O.ref_max_threads()


def _ref(method, prob, **kw):
    p = prob
    plo = p.inputs.lower if p.inputs is not None else None
    phi = p.inputs.upper if p.inputs is not None else None
    return O.ref_reach(method, p.model, p.initial.lower, p.initial.upper, plo, phi, p.t0, p.t1,
                       p.h, p.tube_stride, workers=_need_ref(), **kw)


def _heat_random(g, steps, stride, seed=21):
    n = g ** 3
    rng = np.random.default_rng(seed)
    lo = rng.uniform(0.5, 1.0, n)
    hi = lo + rng.uniform(0.0, 0.5, n)
    m = pk.make_heat3d(g)
    h = BENCH_HKK / (g - 1) ** 2
    return m, pk.ReachProblem(m, pk.IntervalVector(lo, hi), None, 0.0, steps * h, h, stride)


# ------------------------------------------------------------- C5: heat3d

@pytest.mark.parametrize("g,stride", [(200, 0), (200, 5), (400, 0)])
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_heat_bench_ratio_vs_reference(g, stride, mode):
    """heat3d CTMM at g = 200 / 400, 10 RK4 steps at the bench's h*alpha/delta^2,
    random box: exact mode bit-identical to the reference, fast mode within
    1e-12.  Stride 0 with n >= 2^22 in fast mode takes the field-pipelined
    driver the bench's e2e call uses; stride 5 records 3 slots."""
    m, prob = _heat_random(g, 10, stride)
    ref = _ref(O.METHOD_MM, prob)
    c = pk.Context(0, mode)
    try:
        tube = pk.mixed_monotonicity(prob, ctx=c)
    finally:
        c.close()
    if mode == "exact":
        assert_bitexact(tube, ref)
    else:
        assert_within(tube, ref, rel=1e-12)


def _device_heat_uniform(g, steps, h, mode, world=1, K=1):
    """Device-resident heat3d CTMM from the catalog box [0.9, 1.1] (bench.py's
    workload), run through the sharded driver with `world` virtual ranks on
    this GPU.  Returns the owned (lower, upper) slabs as torch tensors."""
    import torch
    from paper_2001_10635_b200 import sharded as S

    m = pk.make_heat3d(g)
    ctx = pk.Context(0, mode)
    runs = []
    try:
        for r in range(world):
            sh = S.Shard(g, world, r, 4 * K)
            run = S.ShardedReach(m, "mixed-monotonicity", sh, S.device_step_fn(m, "mixed-monotonicity", ctx),
                                 None, K=K)
            a = run.alloc(lambda n: torch.empty(n, dtype=torch.float64, device="cuda"))
            a[0].fill_(0.9)
            a[1].fill_(1.1)
            runs.append(run)
        steps_th = S.plan_rk4_steps(0.0, steps * h, h)
        for i, st in enumerate(steps_th):
            if world > 1 and i % K == 0:
                from tests.test_gpu_parity import _fill_halos
                _fill_halos(runs, g * g)
            for run in runs:
                run.run([st], i)
        torch.cuda.synchronize()
        out = [run.owned() for run in runs]
        for run in runs:
            run.b = None
        return out
    finally:
        ctx.close()


def _compare_planes(field, line, g, exact):
    """field: owned slab (planes*g*g) as a torch tensor; every row of g
    components must equal `line` (bit-exact or within 1e-12 relative)."""
    import torch

    ln = torch.from_numpy(line).to(field.device)
    rows = field.view(-1, g)
    worst = 0.0
    for c0 in range(0, rows.shape[0], 1 << 18):
        blk = rows[c0:c0 + (1 << 18)]
        if exact:
            assert bool((blk == ln).all()), f"row block {c0} differs from the 1-D line"
        else:
            rel = ((blk - ln).abs() / ln.abs()).max().item()
            worst = max(worst, rel)
    assert worst <= 1e-12, worst
    return worst


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_c5_full_size_uniform_box(mode):
    """C5 itself: g = 1600 (n = 4.096e9, 131 GB of state), the bench's h and
    box, 8 RK4 steps: every one of the 2n state components equals the exact 1-D
    restatement (bit-identical in exact mode, <= 1e-12 relative in fast mode)."""
    import torch

    g, h, steps = 1600, 5e-8, 8
    (lo, hi), = _device_heat_uniform(g, steps, h, mode)
    try:
        for f, v in ((lo, 0.9), (hi, 1.1)):
            _compare_planes(f, O.heat_line_uniform(g, v, steps, h), g, mode == "exact")
    finally:
        del lo, hi
        torch.cuda.empty_cache()


def test_c5_sharded_three_virtual_ranks_g400():
    """1 GPU == 3 virtual ranks at g = 400 (z-slabs, halo 4, exchange every
    step, interior/boundary split), exact mode, against the exact line."""
    import torch

    g, steps = 400, 6
    h = BENCH_HKK / (g - 1) ** 2
    parts = _device_heat_uniform(g, steps, h, "exact", world=3)
    for (lo, hi) in parts:
        _compare_planes(lo, O.heat_line_uniform(g, 0.9, steps, h), g, True)
        _compare_planes(hi, O.heat_line_uniform(g, 1.1, steps, h), g, True)
    del parts
    torch.cuda.empty_cache()


def test_c5_sharded_three_virtual_ranks_g400_random_box():
    """Same split with a random box (no plane symmetry): the 3-rank result is
    bit-identical to the single-device full-domain reach."""
    import torch
    from paper_2001_10635_b200 import sharded as S
    from tests.test_gpu_parity import _NoopExchanger, _fill_halos

    g, steps = 400, 4
    m, prob = _heat_random(g, steps, 0, seed=4)
    c = pk.Context(0, "exact")
    try:
        ref = pk.mixed_monotonicity(prob, ctx=c).entries[-1].box
        unit = g * g
        lo, hi = prob.initial.lower, prob.initial.upper
        runs = []
        for r in range(3):
            sh = S.Shard(g, 3, r, 4)
            run = S.ShardedReach(m, "mixed-monotonicity", sh, S.device_step_fn(m, "mixed-monotonicity", c),
                                 _NoopExchanger(), K=1)
            run.alloc(lambda k: torch.empty(k, dtype=torch.float64, device="cuda"))
            sl = slice(sh.win_begin * unit, sh.win_end * unit)
            run.a[0].copy_(torch.from_numpy(np.ascontiguousarray(lo[sl])))
            run.a[1].copy_(torch.from_numpy(np.ascontiguousarray(hi[sl])))
            runs.append(run)
        for i, st in enumerate(S.plan_rk4_steps(0.0, prob.t1, prob.h)):
            _fill_halos(runs, unit)
            for run in runs:
                run.run([st], i)
        torch.cuda.synchronize()
        for run in runs:
            o0, o1 = run.owned()
            b, e = run.shard.begin * unit, run.shard.end * unit
            assert np.array_equal(o0.cpu().numpy(), ref.lower[b:e])
            assert np.array_equal(o1.cpu().numpy(), ref.upper[b:e])
    finally:
        c.close()
        torch.cuda.empty_cache()


# --------------------------------------------------- C3: traffic n = 1e6

# values the reference itself produces (bit-stable at -O2/-O3,
# workers 1/8) for traffic CTMM n = 1e6, 60 steps, box [10, 20], p in [4, 6]
C3_GOLD = (8.4261226388996242, 15.671837256973982, 8.8249690258461371)


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_c3_traffic_n1e6_vs_reference(mode):
    n = 10 ** 6
    m = pk.make_traffic(n)
    prob = pk.ReachProblem(m, pk.IntervalVector(np.full(n, 10.0), np.full(n, 20.0)),
                           pk.IntervalVector([4.0], [6.0]), 0.0, 30.0, 0.5, 10)
    ref = _ref(O.METHOD_MM, prob)
    assert (ref.lower[-1][0], ref.upper[-1][0], ref.lower[-1][-1]) == C3_GOLD
    c = pk.Context(0, mode)
    try:
        tube = pk.mixed_monotonicity(prob, ctx=c)
        gb = pk.growth_bound(prob, ctx=c)
    finally:
        c.close()
    ref_gb = _ref(O.METHOD_GB, prob)
    if mode == "exact":
        assert_bitexact(tube, ref)
        assert_bitexact(gb, ref_gb)
        fin = tube.entries[-1].box
        assert (fin.lower[0], fin.upper[0], fin.lower[-1]) == C3_GOLD
    else:
        assert_within(tube, ref, rel=1e-12)
        assert_within(gb, ref_gb, rel=1e-12)


# ------------------------------------------------- C4: coupled chain n = 1e7

def test_c4_chain_n1e7_100_steps_exact():
    """SURVEY.md 8(d) C4 at full size: n = 1e7, h = 0.01, 100 steps, stride 10
    (11 slots), centres 2*u01(7,0,i)-1, half-width 0.05, input [-0.1, 0.1];
    bit-identical to the reference's mixed_monotonicity on the same lambdas."""
    n = 10 ** 7
    ctr = 2.0 * _u01_vec(7, 0, n) - 1.0
    m = pk.make_chain(n)
    prob = pk.ReachProblem(m, pk.IntervalVector(ctr - 0.05, ctr + 0.05), pk.IntervalVector([-0.1], [0.1]),
                           0.0, 1.0, 0.01, 10)
    ref = _ref(O.METHOD_MM, prob)
    c = pk.Context(0, "exact")
    try:
        tube = pk.mixed_monotonicity(prob, ctx=c)
    finally:
        c.close()
    assert len(tube.entries) == 11
    assert_bitexact(tube, ref)


def test_c4_chain_n1e7_fast():
    n = 10 ** 7
    ctr = 2.0 * _u01_vec(7, 0, n) - 1.0
    m = pk.make_chain(n)
    prob = pk.ReachProblem(m, pk.IntervalVector(ctr - 0.05, ctr + 0.05), pk.IntervalVector([-0.1], [0.1]),
                           0.0, 1.0, 0.01, 0)
    ref = _ref(O.METHOD_MM, prob)
    c = pk.Context(0, "fast")
    try:
        tube = pk.mixed_monotonicity(prob, ctx=c)
    finally:
        c.close()
    # the chain's bounds pass through zero: relative 1e-12 plus 1e-15 absolute
    assert_within(tube, ref, rel=1e-12, atol=1e-15)


def _u01_vec(seed, stream, n):
    out = O.u01_vec(seed, stream, np.arange(n, dtype=np.uint64))
    assert all(out[k] == O.u01(seed, stream, k) for k in (0, 1, 2, n // 3, n - 1))
    return out


# ------------------------------------------------------- C2: Monte Carlo m = 1e6

def test_c2_arch_quad_mc_m1e6_vs_reference():
    """C2 at full size: arch-quadrotor, m = 1e6 samples, seed 1, 100 steps,
    stride 10; CUDA sin/cos vs glibc -> relative 1e-12 (+1e-14 absolute near 0)."""
    m = pk.make_arch_quadrotor()
    lo = np.array([-0.4] * 6 + [0.0] * 6)
    prob = pk.ReachProblem(m, pk.IntervalVector(lo, -lo), None, 0.0, 1.0, 0.01, 10)
    ref = _ref(O.METHOD_MC, prob, samples=10 ** 6, seed=1)
    for mode in ("exact", "fast"):
        c = pk.Context(0, mode)
        try:
            tube = pk.monte_carlo(prob, pk.MonteCarloSpec(seed=1, samples_override=10 ** 6), ctx=c)
        finally:
            c.close()
        assert tube.report.m == 10 ** 6
        assert_within(tube, ref, rel=1e-12, atol=1e-14)


def test_c2_laub_loomis_mc_m1e6_bitexact():
    m = pk.make_laub_loomis()
    c = np.array([1.2, 1.05, 1.5, 2.4, 1.0, 0.1, 0.45])
    prob = pk.ReachProblem(m, pk.IntervalVector(c - 0.05, c + 0.05), None, 0.0, 1.0, 0.005, 20)
    ref = _ref(O.METHOD_MC, prob, samples=10 ** 6, seed=1)
    ctx = pk.Context(0, "exact")
    try:
        tube = pk.monte_carlo(prob, pk.MonteCarloSpec(seed=1, samples_override=10 ** 6), ctx=ctx)
    finally:
        ctx.close()
    assert_bitexact(tube, ref)
