"""CPU, multi-process (gloo): the sharded driver used for N > 1 GPUs.

Each rank runs paper_2001_10635_b200.sharded.ShardedReach on its slab with
deep halos exchanged by HaloExchanger (torch.distributed point-to-point),
exactly as on NCCL; here the per-step executor is the oracle's windowed RK4
step (test infrastructure), which reads NaN outside its window so any halo
bug poisons the result.  The gathered result must be bit-identical to the
single-process oracle run (SURVEY.md 8e invariant: k-GPU == 1-GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2001_10635_b200 as pk
from oracle import oracle as O
from paper_2001_10635_b200 import sharded as S


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_step_fn(model, method):
    meth = 0 if method == "mixed-monotonicity" else 1
    unit = S.units_of(model)[1]

    def step(in0, in1, out0, out1, wb, wl, lo, hi, p0, p1, t, hk, k, fail_ptr=0):
        o0, o1 = O.step_window(model, meth, in0.numpy(), in1.numpy(), wb, wl, lo, hi, p0, p1, t,
                               hk)
        a = (lo - wb) * unit
        out0[a:a + o0.size] = torch.from_numpy(o0)
        out1[a:a + o1.size] = torch.from_numpy(o1)
    return step


def problem(kind):
    if kind == "traffic":
        m = pk.make_traffic(301)
        lo = 10.0 + (np.arange(301) % 7)
        return m, "mixed-monotonicity", lo, lo + 5.0, [4.0], [6.0], 0.0, 6.0, 0.5
    if kind == "traffic_gb":
        m = pk.make_traffic(301)
        lo = 10.0 + (np.arange(301) % 7)
        return m, "growth-bound", lo, lo + 5.0, [4.0], [6.0], 0.0, 6.0, 0.5
    if kind == "chain":
        m = pk.make_chain(257)
        c = 2.0 * np.array([O.u01(7, 0, i) for i in range(257)]) - 1.0
        return m, "mixed-monotonicity", c - 0.05, c + 0.05, [-0.1], [0.1], 0.0, 0.1, 0.01
    m = pk.make_heat3d(26)
    n = m.dim
    lo = 0.9 - 0.05 * ((np.arange(n) * 7) % 5)
    return m, "mixed-monotonicity", lo, lo + 0.2, None, None, 0.0, 0.003, 0.0003


def worker(rank, world, port, kind, K, q, overlap=True):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, method, lo, hi, plo, phi, t0, t1, h = problem(kind)
        units, unit = S.units_of(m)
        shard = S.Shard(units, world, rank, 4 * K)
        if method == "growth-bound":
            c0, r0 = 0.5 * (hi + lo), 0.5 * (hi - lo)
            p0 = [0.5 * (phi[0] + plo[0])]
            p1 = [0.5 * (phi[0] - plo[0])]
            f0, f1 = c0, r0
        else:
            f0, f1, p0, p1 = lo, hi, plo, phi
        ex = S.HaloExchanger(shard, unit)
        run = S.ShardedReach(m, method, shard, oracle_step_fn(m, method), ex, p0, p1, K=K)
        a = run.alloc(lambda n: torch.full((n,), float("nan"), dtype=torch.float64))
        sl = slice(shard.win_begin * unit, shard.win_end * unit)
        a[0].copy_(torch.from_numpy(np.ascontiguousarray(f0[sl])))
        a[1].copy_(torch.from_numpy(np.ascontiguousarray(f1[sl])))
        run.run(S.plan_rk4_steps(t0, t1, h), 0, overlap=overlap)
        o0, o1 = run.owned()
        q.put((rank, shard.begin * unit, o0.numpy().copy(), o1.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,world,K,overlap", [("traffic", 2, 1, True), ("traffic", 3, 2, True),
                                                  ("chain", 2, 1, True), ("chain", 3, 3, True),
                                                  ("heat", 2, 1, True), ("heat", 3, 1, True),
                                                  ("traffic_gb", 2, 2, True), ("heat", 2, 1, False),
                                                  ("chain", 3, 2, False)])
def test_sharded_equals_single(kind, world, K, overlap):
    """k-rank results are bit-identical to the single-device oracle, with the
    halo exchange overlapped with the interior step (overlap=True) or not."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, kind, K, q, overlap)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m, method, lo, hi, plo, phi, t0, t1, h = problem(kind)
    fn = O.mixed_monotonicity if method == "mixed-monotonicity" else O.growth_bound
    ref = fn(m, lo, hi, plo, phi, t0, t1, h, 0)
    n = m.dim
    g0 = np.full(n, np.nan)
    g1 = np.full(n, np.nan)
    for _, off, o0, o1 in parts:
        g0[off:off + o0.size] = o0
        g1[off:off + o1.size] = o1
    if method == "growth-bound":  # box epilogue (reach.cpp:121-134)
        r = np.where((g1 < 0) & (g1 >= -1e-12), 0.0, g1)
        g0, g1 = g0 - r, g0 + r
    assert np.array_equal(g0, ref.lower[-1]) and np.array_equal(g1, ref.upper[-1])


def mc_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = pk.make_laub_loomis()
        c = np.array([1.2, 1.05, 1.5, 2.4, 1.0, 0.1, 0.45])
        s0, s1 = S.mc_sample_range(1000, world, rank)
        r = O.monte_carlo(m, c - 0.05, c + 0.05, None, None, 0.0, 0.5, 0.005, 20, 9, 1000, s0, s1)
        lo, hi = torch.from_numpy(r.lower.copy()), torch.from_numpy(r.upper.copy())
        S.allreduce_hull(lo, hi)
        q.put((rank, lo.numpy(), hi.numpy()))
    finally:
        dist.destroy_process_group()


def test_mc_sample_sharding_allreduce():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=mc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    m = pk.make_laub_loomis()
    c = np.array([1.2, 1.05, 1.5, 2.4, 1.0, 0.1, 0.45])
    ref = O.monte_carlo(m, c - 0.05, c + 0.05, None, None, 0.0, 0.5, 0.005, 20, 9, 1000)
    for _, lo, hi in parts:
        assert np.array_equal(lo, ref.lower) and np.array_equal(hi, ref.upper)


def test_shard_geometry():
    for units, world, halo in [(1600, 8, 4), (1000, 3, 8), (26, 3, 4)]:
        covered = []
        for r in range(world):
            s = S.Shard(units, world, r, halo)
            assert s.win_begin <= s.begin < s.end <= s.win_end
            lo, hi = s.out_range(halo // 4 - 1)
            assert lo <= s.begin and hi >= s.end
            covered.extend(range(s.begin, s.end))
        assert covered == list(range(units))


def test_bench_gpus_flag_launches_n_ranks():
    """`python bench.py --gpus 2` re-executes itself under torch.distributed.run
    with two ranks (--gpus was parsed and ignored)."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--launcher-check"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert sorted(l["rank"] for l in lines) == [0, 1]
    assert all(l["world"] == 2 and l["n_gpus"] == 2 for l in lines)
    # a WORLD_SIZE that disagrees with --gpus is refused
    env2 = dict(env, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r2 = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--launcher-check"],
                        cwd=root, env=env2, capture_output=True, text=True, timeout=120)
    assert r2.returncode != 0 and "WORLD_SIZE=3" in r2.stderr


class _LockstepPeers(S.PeerStores):
    """PeerStores with the transport replaced for a one-process CPU check of
    ShardedReach._run_peer: "peer memory" is the neighbour rank's window tensor
    (a view), flags are recorded.  Ranks are stepped one after another per RK4
    step, which is an order the real flags allow."""

    def __init__(self, shard, unit):
        self.shard, self.unit, self.seq = shard, unit, 0
        self.waits, self.signals = [], []

    def link(self, runs):
        s = self.shard
        self.local = [runs[s.rank].a[0], runs[s.rank].a[1], runs[s.rank].b[0], runs[s.rank].b[1]]
        self.nb = {}
        for side, r in (("left", s.rank - 1), ("right", s.rank + 1)):
            if 0 <= r < s.world:
                o = runs[r]
                self.nb[side] = {"win_begin": o.shard.win_begin, "bufs": [o.a[0], o.a[1], o.b[0], o.b[1]]}

    def wait(self, value):
        self.waits.append(value)

    def signal(self, value):
        self.signals.append(value)

    def _target(self, side, idx, out_begin):
        nb = self.nb[side]
        return nb["bufs"][idx], out_begin - nb["win_begin"]


@pytest.mark.parametrize("kind,world,fused", [("traffic", 2, True), ("traffic", 3, True), ("chain", 4, True),
                                              ("heat", 2, True), ("heat", 3, True), ("traffic_gb", 2, True),
                                              ("traffic", 3, False), ("heat", 3, False), ("chain", 4, False)])
def test_peer_store_schedule_equals_single(kind, world, fused):
    """The peer-store schedules (fused: one launch per slab storing its edge
    units into the neighbours' windows; split: boundary units first, then the
    interior) with the oracle's windowed step, which reads NaN outside its
    window: bit-identical to one process, and the flag protocol waits for k-1
    before raising k on every step."""
    m, method, lo, hi, plo, phi, t0, t1, h = problem(kind)
    units, unit = S.units_of(m)
    if method == "growth-bound":
        f0, f1 = 0.5 * (hi + lo), 0.5 * (hi - lo)
        p0, p1 = [0.5 * (phi[0] + plo[0])], [0.5 * (phi[0] - plo[0])]
    else:
        f0, f1, p0, p1 = lo, hi, plo, phi
    base = oracle_step_fn(m, method)

    def step(in0, in1, out0, out1, wb, wl, lo_, hi_, p0_, p1_, t, hk, k, fail_ptr=0, mirror=None):
        base(in0, in1, out0, out1, wb, wl, lo_, hi_, p0_, p1_, t, hk, k)
        if mirror is None:
            return
        lo0, lo1, lo_end, hi0, hi1, hi_begin = mirror

        def put(t0, t1, u0, u1):  # units [u0, u1) into the target pair
            if t0 is None or u0 >= u1:
                return
            (d0, off), (d1, _) = t0, t1
            a, n, b = (u0 - wb) * unit, (u1 - u0) * unit, (u0 - lo_ + off) * unit
            assert b >= 0
            d0[b:b + n] = out0[a:a + n]
            d1[b:b + n] = out1[a:a + n]
        put(lo0, lo1, lo_, min(hi_, lo_end))
        put(hi0, hi1, max(lo_, hi_begin), hi_)

    runs, exs = [], []
    for r in range(world):
        shard = S.Shard(units, world, r, 4)
        ex = _LockstepPeers(shard, unit)
        ex.fused = fused
        run = S.ShardedReach(m, method, shard, step, ex, p0, p1, K=1)
        a = run.alloc(lambda n: torch.full((n,), float("nan"), dtype=torch.float64))
        sl = slice(shard.win_begin * unit, shard.win_end * unit)
        a[0].copy_(torch.from_numpy(np.ascontiguousarray(f0[sl])))
        a[1].copy_(torch.from_numpy(np.ascontiguousarray(f1[sl])))
        # halos of the second buffer stay NaN: only peer stores may fill them
        runs.append(run)
        exs.append(ex)
    for ex in exs:
        ex.link(runs)
    plan = S.plan_rk4_steps(t0, t1, h)
    for k, st in enumerate(plan):
        for run in runs:
            run.run([st], k)
    got0 = np.concatenate([run.owned()[0].numpy() for run in runs])
    got1 = np.concatenate([run.owned()[1].numpy() for run in runs])
    meth = 0 if method == "mixed-monotonicity" else 1
    # single-process reference: the same oracle step over the whole state
    a0, a1 = f0.copy(), f1.copy()
    for t, hk in plan:
        a0, a1 = O.step_window(m, meth, a0, a1, 0, units, 0, units, p0, p1, t, hk)
    np.testing.assert_array_equal(got0, a0)
    np.testing.assert_array_equal(got1, a1)
    for ex in exs:
        assert ex.waits == list(range(len(plan)))
        assert ex.signals == list(range(1, len(plan) + 1))
