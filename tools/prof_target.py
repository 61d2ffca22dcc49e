"""Run a few engine steps of one configuration (target for ncu)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_10635_b200 as pk

which, size, mode, steps = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
ctx = pk.Context(0, mode)
if which == "heat":
    m = pk.make_heat3d(size); n = size ** 3
    prob = pk.ReachProblem(m, pk.IntervalVector(np.full(n, 0.9), np.full(n, 1.1)), None, 0.0, 100 * 5e-8, 5e-8, 0)
elif which == "traffic":
    m = pk.make_traffic(size); n = size
    prob = pk.ReachProblem(m, pk.IntervalVector(np.full(n, 10.0), np.full(n, 20.0)), pk.IntervalVector([4.0], [6.0]), 0.0, 30.0, 0.5, 0)
else:
    m = pk.make_chain(size); n = size
    prob = pk.ReachProblem(m, pk.IntervalVector(np.full(n, -0.05), np.full(n, 0.05)), pk.IntervalVector([-0.1], [0.1]), 0.0, 1.0, 0.01, 0)
eng = pk.Engine(prob, ctx=ctx)
eng.advance(steps)
print("done", eng.status())
