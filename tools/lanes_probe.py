"""Overhead of the multi-lane (sharded) driver on one GPU: heat3d CTMM through
pirk_mixed_monotonicity with 1, 2, 4 and 8 lanes on cuda:0 (dev probe).  The
integration phase of the report is compared; same results by construction."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_10635_b200 as pk

g = int(sys.argv[1]) if len(sys.argv) > 1 else 800
mode = sys.argv[2] if len(sys.argv) > 2 else "fast"
steps = 20
n = g ** 3
m = pk.make_heat3d(g)
h = 5e-8 * (1599.0 / (g - 1)) ** 2
lo = np.full(n, 0.9)
hi = np.full(n, 1.1)
prob = pk.ReachProblem(m, pk.IntervalVector(lo, hi, validate=False), None, 0.0, steps * h, h, 0)
out = (np.empty(n), np.empty(n))
for lanes in (1, 2, 4, 8):
    ctx = pk.Context(devices=[0] * lanes, mode=mode)
    os.environ["PIRK_PIPELINE"] = "0"
    pk.mixed_monotonicity(prob, ctx=ctx, out=out)
    best = 1e9
    for _ in range(3):
        t = pk.mixed_monotonicity(prob, ctx=ctx, out=out)
        best = min(best, t.report.phases.integration_s)
    print(f"g={g} {mode} lanes={lanes}: integration {best*1e3:.1f} ms for {steps} steps "
          f"({best/steps*1e3:.3f} ms/step incl. final D2H)", flush=True)
    ctx.close()
