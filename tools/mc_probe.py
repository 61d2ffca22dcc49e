"""C2 Monte Carlo timing (arch-quadrotor, m = 1e6, 100 steps) for A/B builds (dev only)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_10635_b200 as pk

mode = sys.argv[1] if len(sys.argv) > 1 else "fast"
ctx = pk.Context(0, mode)
mq = pk.make_arch_quadrotor()
lo = np.array([-0.4] * 6 + [0.0] * 6)
p = pk.ReachProblem(mq, pk.IntervalVector(lo, -lo), None, 0.0, 1.0, 0.01, 0)
pk.monte_carlo(p, pk.MonteCarloSpec(seed=1, samples_override=10 ** 5), ctx=ctx)
best = 1e9
for _ in range(3):
    t0 = time.perf_counter()
    tube = pk.monte_carlo(p, pk.MonteCarloSpec(seed=1, samples_override=10 ** 6), ctx=ctx)
    best = min(best, time.perf_counter() - t0)
print(f"MC arch-quad {mode}: {best * 1e3:.2f} ms  {1e6 * tube.report.steps / best:.3e} sample-steps/s")
