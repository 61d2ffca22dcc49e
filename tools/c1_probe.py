"""C1 timing: arch-quadrotor CTMM (Jacobian decomposition), 100 steps, stride 10 (dev probe)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_10635_b200 as pk

ctx = pk.Context(0, sys.argv[1] if len(sys.argv) > 1 else "exact")
mq = pk.with_jacobian_decomposition(pk.make_arch_quadrotor())
lo = np.array([-0.4] * 6 + [0.0] * 6)
p = pk.ReachProblem(mq, pk.IntervalVector(lo, -lo), None, 0.0, 1.0, 0.01, 10)
pk.mixed_monotonicity(p, ctx=ctx)
t0 = time.perf_counter()
for _ in range(20):
    tube = pk.mixed_monotonicity(p, ctx=ctx)
dt = (time.perf_counter() - t0) / 20
print(f"C1 {'serial' if os.environ.get('PIRK_SMALL_SERIAL') else 'warp'}: call {dt*1e3:.3f} ms, "
      f"kernel+copies {tube.report.phases.integration_s*1e3:.3f} ms")
