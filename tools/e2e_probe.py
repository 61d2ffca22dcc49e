"""C5 end-to-end call timing (the bench's e2e leg) for A/B of the
field-pipelined driver's schedules: run once per environment variant, e.g.
PIRK_SKEW=0 python tools/e2e_probe.py.  Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_10635_b200 as pk  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 1600
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
h = 5e-8
n = g ** 3
bufs = [np.empty(n) for _ in range(4)]
cudart = torch.cuda.cudart()
for b in bufs:
    cudart.cudaHostRegister(b.ctypes.data, b.nbytes, 0)
lo, hi, olo, ohi = bufs
lo.fill(0.9)
hi.fill(1.1)
prob = pk.ReachProblem(pk.make_heat3d(g), pk.IntervalVector(lo, hi), None, 0.0, 100 * h, h, 0)
ctx = pk.get_context(0)
ctx.set_mode("fast")
pk.mixed_monotonicity(prob, ctx=ctx, out=(olo, ohi))
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    tube = pk.mixed_monotonicity(prob, ctx=ctx, out=(olo, ohi))
    ts.append(time.perf_counter() - t0)
chk = float(olo[:: max(1, n // 4096)].sum() + ohi[:: max(1, n // 4096)].sum())
env = {k: v for k, v in os.environ.items() if k.startswith("PIRK_")}
print(json.dumps({"grid": g, "env": env, "seconds": ts, "best": min(ts),
                  "upd_per_s": 2.0 * n * 100 / min(ts), "checksum": chk,
                  "launches": tube.report.kernel_launches}))
