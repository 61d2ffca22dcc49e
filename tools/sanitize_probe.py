"""Small invocations of every product kernel, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Development tool, not a test:

    compute-sanitizer --tool racecheck python tools/sanitize_probe.py heat_fast

Workloads are sized so each kernel runs its interior, edge and chunk paths
(heat: g=130 = 3 tiles of 56 per axis, 2 z-chunks) in a few launches.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2001_10635_b200 as pk  # noqa: E402


def heat(mode, g, steps=2):
    ctx = pk.Context(0, mode)
    n = g ** 3
    m = pk.make_heat3d(g)
    p = pk.ReachProblem(m, pk.IntervalVector(np.full(n, 0.9), np.full(n, 1.1)), None, 0.0,
                        steps * 5e-6, 5e-6, 1)
    t = pk.mixed_monotonicity(p, ctx=ctx)
    assert np.isfinite(t.entries[-1].box.lower).all()
    ctx.close()


def chain(mode, kind, n=5000, steps=4):
    ctx = pk.Context(0, mode)
    if kind == "traffic":
        m = pk.make_traffic(n)
        p = pk.ReachProblem(m, pk.IntervalVector(np.full(n, 10.0), np.full(n, 20.0)),
                            pk.IntervalVector([4.0], [6.0]), 0.0, steps * 0.5, 0.5, 2)
    else:
        m = pk.make_chain(n)
        c = np.linspace(-1, 1, n)
        p = pk.ReachProblem(m, pk.IntervalVector(c - 0.05, c + 0.05),
                            pk.IntervalVector([-0.1], [0.1]), 0.0, steps * 0.01, 0.01, 2)
    pk.mixed_monotonicity(p, ctx=ctx)
    ctx.close()


def mc(mode, m_samples=4096):
    ctx = pk.Context(0, mode)
    mq = pk.make_arch_quadrotor()
    lo = np.array([-0.4] * 6 + [0.0] * 6)
    p = pk.ReachProblem(mq, pk.IntervalVector(lo, -lo), None, 0.0, 0.1, 0.01, 5)
    pk.monte_carlo(p, pk.MonteCarloSpec(seed=1, samples_override=m_samples), ctx=ctx)
    ll = pk.make_laub_loomis()
    c = np.array([1.2, 1.05, 1.5, 2.4, 1.0, 0.1, 0.45])
    p2 = pk.ReachProblem(ll, pk.IntervalVector(c - 0.05, c + 0.05), None, 0.0, 0.1, 0.01, 5)
    pk.monte_carlo(p2, pk.MonteCarloSpec(seed=1, samples_override=m_samples), ctx=ctx)
    ctx.close()


def lanes(mode):
    """Multi-lane context: chain index ranges, heat z-slabs (peer-copy halos,
    cross-lane events) and Monte Carlo sample ranges on 3 lanes of cuda:0."""
    ctx = pk.Context(devices=[0, 0, 0], mode=mode)
    chain_n = 3000
    m = pk.make_traffic(chain_n)
    p = pk.ReachProblem(m, pk.IntervalVector(np.full(chain_n, 10.0), np.full(chain_n, 20.0)),
                        pk.IntervalVector([4.0], [6.0]), 0.0, 2.0, 0.5, 2)
    pk.mixed_monotonicity(p, ctx=ctx)
    pk.growth_bound(p, ctx=ctx)
    g = 40
    hm = pk.make_heat3d(g)
    hp = pk.ReachProblem(hm, pk.IntervalVector(np.full(g ** 3, 0.9), np.full(g ** 3, 1.1)), None, 0.0,
                         3 * 1e-4, 1e-4, 1)
    pk.mixed_monotonicity(hp, ctx=ctx)
    ll = pk.make_laub_loomis()
    c = np.array([1.2, 1.05, 1.5, 2.4, 1.0, 0.1, 0.45])
    p2 = pk.ReachProblem(ll, pk.IntervalVector(c - 0.05, c + 0.05), None, 0.0, 0.1, 0.01, 5)
    pk.monte_carlo(p2, pk.MonteCarloSpec(seed=1, samples_override=3000), ctx=ctx)
    ctx.close()


USER_SRC = r"""
__device__ double pirk_rhs(u64 i, double, const double* x, const double* p) {
    const double l = i > 0 ? x[i - 1] : p[0];
    const double r = i + 1 < PIRK_N ? x[i + 1] : 0.0;
    return 0.5 * (l - x[i]) - 0.25 * (x[i] - r) / (1.0 + x[i] * x[i]);
}
__device__ double pirk_decomposition(u64 i, double t, const double* x, const double* p, const double*,
                                     const double*) { return pirk_rhs(i, t, x, p); }
__device__ double pirk_growth(u64 i, double, const double* r, const double* w) {
    return 0.5 * (i > 0 ? r[i - 1] : w[0]) + 0.25 * (i + 1 < PIRK_N ? r[i + 1] : 0.0);
}
"""


def user(mode):
    """NVRTC user-model kernels: one-thread (n <= 64), per-component stage
    (n > 64) and Monte Carlo, plus the catalog MC beyond 64 components."""
    ctx = pk.Context(0, mode)
    for n in (12, 300):
        m = pk.make_user_model(USER_SRC, n, 1, decomposition=True, growth=True, input_affine=True)
        p = pk.ReachProblem(m, pk.IntervalVector(np.zeros(n), np.ones(n)), pk.IntervalVector([0.5], [1.0]),
                            0.0, 0.2, 0.05, 2)
        pk.mixed_monotonicity(p, ctx=ctx)
        pk.growth_bound(p, ctx=ctx)
        pk.monte_carlo(p, pk.MonteCarloSpec(seed=2, samples_override=700), ctx=ctx)
    tm = pk.make_traffic(100)
    tp = pk.ReachProblem(tm, pk.IntervalVector(np.full(100, 10.0), np.full(100, 20.0)),
                         pk.IntervalVector([4.0], [6.0]), 0.0, 1.0, 0.5, 1)
    pk.monte_carlo(tp, pk.MonteCarloSpec(seed=2, samples_override=500), ctx=ctx)
    ctx.close()


CASES = {
    "lanes_exact": lambda: lanes("exact"),
    "lanes_fast": lambda: lanes("fast"),
    "user_exact": lambda: user("exact"),
    "user_fast": lambda: user("fast"),
    "heat_fast": lambda: heat("fast", 130),
    "heat_exact": lambda: heat("exact", 72),
    "chain_fast": lambda: chain("fast", "chain"),
    "chain_exact": lambda: chain("exact", "chain"),
    "traffic_fast": lambda: chain("fast", "traffic"),
    "traffic_exact": lambda: chain("exact", "traffic"),
    "mc_fast": lambda: mc("fast"),
    "mc_exact": lambda: mc("exact"),
}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        print(f"{name}: done", flush=True)
