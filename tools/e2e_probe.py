"""C5 end-to-end reach timing (pinned host buffers, H2D + 100 steps + D2H) for A/B builds (dev only)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2001_10635_b200 as pk

g = int(sys.argv[1]) if len(sys.argv) > 1 else 1600
n = g ** 3
lo = torch.full((n,), 0.9, dtype=torch.float64).pin_memory()
hi = torch.full((n,), 1.1, dtype=torch.float64).pin_memory()
olo = torch.empty((1, n), dtype=torch.float64).pin_memory()
ohi = torch.empty((1, n), dtype=torch.float64).pin_memory()
ctx = pk.Context(0, "fast")
prob = pk.ReachProblem(pk.make_heat3d(g), pk.IntervalVector(lo.numpy(), hi.numpy(), validate=False), None,
                       0.0, 100 * 5e-8, 5e-8, 0)
for r in range(int(os.environ.get("REPS", "2"))):
    t = time.perf_counter()
    tube = pk.mixed_monotonicity(prob, ctx=ctx, out=(olo.numpy(), ohi.numpy()))
    dt = time.perf_counter() - t
    ph = tube.report.phases
    print(f"e2e g={g}: {dt:.3f} s  {2 * n * 100 / dt:.3e} upd/s  (setup {ph.setup_s:.3f} s, integration {ph.integration_s:.3f} s)")
