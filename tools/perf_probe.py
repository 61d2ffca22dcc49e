"""Quick device timing of the engine kernels (development probe, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2001_10635_b200 as pk

def run(name, prob, mode, steps):
    ctx = pk.Context(0, mode)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    eng = pk.Engine(prob, ctx=ctx)
    eng.advance(2); eng.status()
    with torch.cuda.stream(stream):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        eng.advance(steps)
        e.record(stream)
    e.synchronize()
    ms = s.elapsed_time(e) / steps
    n = prob.model.dim
    ups = 2 * n / (ms * 1e-3)
    print(f"{name:28s} {mode:5s} n={n:>12d} {ms:9.4f} ms/step  {ups:.3e} upd/s  "
          f"{ups*16/1e9:8.1f} GB/s  frac={ups*16/6552.3e9:.3f}", flush=True)
    eng.close(); ctx.close()

g = int(sys.argv[1]) if len(sys.argv) > 1 else 400
# PROBE_MODES=fast|exact|exact,fast; PROBE=heat|chain|all (default all)
modes = os.environ.get("PROBE_MODES", "exact,fast").split(",")
what = os.environ.get("PROBE", "all")
for mode in modes:
    if what in ("all", "heat"):
        m = pk.make_heat3d(g)
        n = g ** 3
        prob = pk.ReachProblem(m, pk.IntervalVector(np.full(n, 0.9), np.full(n, 1.1)), None, 0.0, 100 * 5e-8, 5e-8, 0)
        run(f"heat3d g={g}", prob, mode, 20)
    if what == "heat":
        continue
    n6 = 10**6
    m = pk.make_traffic(n6)
    prob = pk.ReachProblem(m, pk.IntervalVector(np.full(n6, 10.0), np.full(n6, 20.0)), pk.IntervalVector([4.0], [6.0]), 0.0, 30.0, 0.5, 0)
    run("traffic n=1e6", prob, mode, 60)
    m = pk.make_traffic(10**7)
    prob = pk.ReachProblem(m, pk.IntervalVector(np.full(10**7, 10.0), np.full(10**7, 20.0)), pk.IntervalVector([4.0], [6.0]), 0.0, 30.0, 0.5, 0)
    run("traffic n=1e7", prob, mode, 20)
    m = pk.make_chain(10**7)
    c = np.zeros(10**7)
    prob = pk.ReachProblem(m, pk.IntervalVector(c - 0.05, c + 0.05), pk.IntervalVector([-0.1], [0.1]), 0.0, 1.0, 0.01, 0)
    run("chain n=1e7", prob, mode, 20)
