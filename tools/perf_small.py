"""Timing of the MC (C2) and chain (C4) paths (development probe)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2001_10635_b200 as pk

for mode in ("exact", "fast"):
    ctx = pk.Context(0, mode)
    m = pk.make_arch_quadrotor(); lo = np.array([-0.4] * 6 + [0.0] * 6)
    p = pk.ReachProblem(m, pk.IntervalVector(lo, -lo), None, 0.0, 1.0, 0.01, 0)
    pk.monte_carlo(p, pk.MonteCarloSpec(seed=1, samples_override=10 ** 5), ctx=ctx)
    t = pk.monte_carlo(p, pk.MonteCarloSpec(seed=1, samples_override=10 ** 6), ctx=ctx)
    print(f"MC arch-quad m=1e6 {mode}: kernel {t.report.phases.integration_s*1e3:.3f} ms -> "
          f"{1e8 / t.report.phases.integration_s:.3e} sample-steps/s", flush=True)
    ll = pk.make_laub_loomis(); c = np.array([1.2, 1.05, 1.5, 2.4, 1.0, 0.1, 0.45])
    p2 = pk.ReachProblem(ll, pk.IntervalVector(c - 0.05, c + 0.05), None, 0.0, 1.0, 0.005, 0)
    t = pk.monte_carlo(p2, pk.MonteCarloSpec(seed=1, samples_override=10 ** 6), ctx=ctx)
    print(f"MC laub-loomis m=1e6 x200 {mode}: kernel {t.report.phases.integration_s*1e3:.3f} ms -> "
          f"{2e8 / t.report.phases.integration_s:.3e} sample-steps/s", flush=True)
    ctx.close()
