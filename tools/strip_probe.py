"""Cost of covering one heat3d RK4 step with z-strips of W planes (2-field
windowed launches through pirk_step_window) -- the per-launch overhead the
skewed e2e schedule pays.  Prints one JSON line per W."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_10635_b200 as pk  # noqa: E402
from paper_2001_10635_b200.reach import step_window  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 1600
widths = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1600", "800", "400", "200", "100", "50"])]
m = pk.make_heat3d(g)
ctx = pk.Context(0, "fast")
n = g ** 3
a0 = torch.full((n,), 0.9, dtype=torch.float64, device="cuda")
a1 = torch.full((n,), 1.1, dtype=torch.float64, device="cuda")
b0 = torch.empty_like(a0)
b1 = torch.empty_like(a1)
s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
unit = g * g
h = 5e-8


def cover(W):
    for lo in range(0, g, W):
        hi = min(g, lo + W)
        step_window(m, "mixed-monotonicity", a0.data_ptr(), a1.data_ptr(), b0.data_ptr() + lo * unit * 8,
                    b1.data_ptr() + lo * unit * 8, 0, g, lo, hi, None, None, 0.0, h, 0, 0, ctx=ctx)


for W in widths:
    for _ in range(2):
        cover(W)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record(s)
    for _ in range(reps):
        cover(W)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"g": g, "W": W, "launches": (g + W - 1) // W, "ms_per_step": ms,
                      "zchunks_env": os.environ.get("PIRK_HEAT_ZCHUNKS")}), flush=True)
