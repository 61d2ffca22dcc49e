"""One process per GPU with peer-store halos (sharded.PeerStores): real CUDA
IPC mappings, cuStreamWaitValue32 flags and the mirror instantiations of the
step kernels, with 2-3 processes on cuda:0 (the only GPU of the test box;
the stores are then device-local but take the same path as over NVLink).
The gathered state must be bit-identical to the oracle's single-process run
in exact mode and within the fast-mode tolerance otherwise."""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(kind):
    import paper_2001_10635_b200 as pk

    if kind == "traffic":
        m = pk.make_traffic(4001)
        lo = 10.0 + (np.arange(4001) % 7)
        return m, "mixed-monotonicity", lo, lo + 5.0, [4.0], [6.0], 0.0, 3.0, 0.5
    if kind == "chain":
        m = pk.make_chain(3001)
        c = 2.0 * np.array([O.u01(7, 0, i) for i in range(3001)]) - 1.0
        return m, "mixed-monotonicity", c - 0.05, c + 0.05, [-0.1], [0.1], 0.0, 0.05, 0.01
    if kind == "traffic_gb":  # fields (center, radius), inputs (center, half-width)
        m = pk.make_traffic(2003)
        c = 12.0 + (np.arange(2003) % 5)
        return m, "growth-bound", c, np.full(2003, 2.5), [5.0], [1.0], 0.0, 2.5, 0.5
    m = pk.make_heat3d(40)
    n = m.dim
    lo = 0.9 - 0.05 * ((np.arange(n) * 7) % 5)
    return m, "mixed-monotonicity", lo, lo + 0.2, None, None, 0.0, 0.002, 0.0003


def _worker(rank, world, port, kind, mode, q, fused=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_2001_10635_b200 as pk
    from paper_2001_10635_b200 import sharded as S

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        m, method, f0, f1, p0, p1, t0, t1, h = _problem(kind)
        units, unit = S.units_of(m)
        ctx = pk.Context(0, mode)
        shard = S.Shard(units, world, rank, 4)
        ex = S.PeerStores(shard, unit, ctx, fused=fused)
        run = S.ShardedReach(m, method, shard, S.device_step_fn(m, method, ctx), ex, p0, p1, K=1)
        dev = torch.device("cuda", 0)
        fail = torch.full((2,), -1, dtype=torch.int64, device=dev)
        a = run.alloc(lambda n: torch.full((n,), float("nan"), dtype=torch.float64, device=dev), fail=fail)
        sl = slice(shard.win_begin * unit, shard.win_end * unit)
        a[0].copy_(torch.from_numpy(np.ascontiguousarray(f0[sl])))
        a[1].copy_(torch.from_numpy(np.ascontiguousarray(f1[sl])))
        ex.attach(run)  # the other buffer's halos stay NaN until peer stores fill them
        plan = S.plan_rk4_steps(t0, t1, h)
        stream = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(stream):
            run.run(plan[:2], 0)  # two calls: the flag sequence continues across runs
            run.run(plan[2:], 2)
        torch.cuda.synchronize()
        run.check(t0, h)
        o0, o1 = run.owned()
        q.put((rank, o0.cpu().numpy(), o1.cpu().numpy(), ex.seq))
        ex.close()
        ctx.close()
    except Exception as e:  # surface the failure in the parent
        q.put((rank, None, repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,world,mode,fused", [("heat", 2, "exact", True), ("heat", 3, "fast", True),
                                                   ("traffic", 3, "exact", True), ("chain", 4, "exact", True),
                                                   ("traffic_gb", 2, "exact", True), ("heat", 2, "fast", True),
                                                   ("heat", 3, "fast", False), ("heat", 3, "exact", False),
                                                   ("chain", 3, "exact", False)])
def test_peer_store_processes_equal_single(kind, world, mode, fused):
    import torch.multiprocessing as mp

    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, world, port, kind, mode, q, fused)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, g0, g1, seq = q.get(timeout=600)
            assert g0 is not None, f"rank {r}: {g1}"
            res[r] = (g0, g1, seq)
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    m, method, f0, f1, p0, p1, t0, t1, h = _problem(kind)
    from paper_2001_10635_b200 import sharded as S

    units, _ = S.units_of(m)
    plan = S.plan_rk4_steps(t0, t1, h)
    meth = 0 if method == "mixed-monotonicity" else 1
    a0, a1 = f0.copy(), f1.copy()
    for t, hk in plan:
        a0, a1 = O.step_window(m, meth, a0, a1, 0, units, 0, units, p0, p1, t, hk)
    got0 = np.concatenate([res[r][0] for r in range(world)])
    got1 = np.concatenate([res[r][1] for r in range(world)])
    assert all(res[r][2] == len(plan) for r in range(world))
    if mode == "exact":
        np.testing.assert_array_equal(got0, a0)
        np.testing.assert_array_equal(got1, a1)
    else:
        for g, ref in ((got0, a0), (got1, a1)):
            assert np.isfinite(g).all()
            assert np.max(np.abs(g - ref) / np.maximum(np.abs(ref), 1e-300)) <= 1e-12
