"""Per-step device time of one rank's heat3d slab (g=1600, N ranks) under the
peer-store schedules, on one GPU with local stand-ins for the neighbours'
windows: fused (one launch, edge planes also stored to both neighbours),
split (two 4-plane boundary launches + interior), and a plain launch."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_10635_b200 as pk  # noqa: E402
from paper_2001_10635_b200 import sharded as S  # noqa: E402
from paper_2001_10635_b200.reach import step_window  # noqa: E402

g = 1600
unit = g * g
m = pk.make_heat3d(g)
ctx = pk.Context(0, "fast")
st = torch.cuda.Stream()
ctx.set_stream(st.cuda_stream)
h = 5e-8
for N in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["8", "4", "2"])]:
    r = N // 2 if N > 1 else 0  # a middle rank: two neighbours
    sh = S.Shard(g, N, r, 4)
    L, R = S.Shard(g, N, r - 1, 4), S.Shard(g, N, r + 1, 4)
    n = sh.win_len * unit
    a = [torch.full((n,), v, dtype=torch.float64, device="cuda") for v in (0.9, 1.1)]
    b = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
    nl = [torch.empty(L.win_len * unit, dtype=torch.float64, device="cuda") for _ in range(2)]
    nr = [torch.empty(R.win_len * unit, dtype=torch.float64, device="cuda") for _ in range(2)]
    wb, wl = sh.win_begin, sh.win_len

    def launch(lo, hi, mirror=None):
        off = (lo - wb) * unit * 8
        step_window(m, "mixed-monotonicity", a[0].data_ptr(), a[1].data_ptr(), b[0].data_ptr() + off,
                    b[1].data_ptr() + off, wb, wl, lo, hi, None, None, 0.0, h, 0, 0, ctx=ctx, mirror=mirror)

    def tgt(t, sh2, lo):
        return t.data_ptr() + (lo - sh2.win_begin) * unit * 8

    def fused():
        launch(sh.begin, sh.end, (tgt(nl[0], L, sh.begin), tgt(nl[1], L, sh.begin), sh.begin + 4,
                                  tgt(nr[0], R, sh.begin), tgt(nr[1], R, sh.begin), sh.end - 4))

    def split():
        launch(sh.begin, sh.begin + 4, (tgt(nl[0], L, sh.begin), tgt(nl[1], L, sh.begin), sh.begin + 4,
                                        None, None, 0))
        launch(sh.end - 4, sh.end, (None, None, 0, tgt(nr[0], R, sh.end - 4), tgt(nr[1], R, sh.end - 4),
                                    sh.end - 4))
        launch(sh.begin + 4, sh.end - 4)

    def plain():
        launch(sh.begin, sh.end)

    res = {"N": N, "planes": sh.end - sh.begin}
    for name, fn in (("plain", plain), ("fused", fused), ("split", split), ("plain2", plain)):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(5):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        res[name + "_ms"] = e0.elapsed_time(e1) / 5
    res["ideal_ms"] = 33.72 * (sh.end - sh.begin) / g
    # correctness of the stand-in stores: the neighbours' halo planes equal the slab's edge planes
    fused()
    torch.cuda.synchronize()
    o = (sh.begin - wb) * unit
    lo_ok = torch.equal(nl[0][(sh.begin - L.win_begin) * unit:(sh.begin - L.win_begin + 4) * unit], b[0][o:o + 4 * unit])
    e = (sh.end - 4 - wb) * unit
    hi_ok = torch.equal(nr[1][(sh.end - 4 - R.win_begin) * unit:(sh.end - R.win_begin) * unit], b[1][e:e + 4 * unit])
    res["stores_ok"] = bool(lo_ok and hi_ok)
    print(json.dumps(res), flush=True)
    del a, b, nl, nr
    torch.cuda.empty_cache()
