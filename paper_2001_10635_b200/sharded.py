"""State-sharded (multi-GPU) mixed-monotonicity / growth-bound runs and
sample-sharded Monte Carlo, one process per GPU.

* 1-D chains (traffic, coupled chain) shard contiguous component ranges;
  heat3d shards contiguous z-slabs (``i = ix + g*iy + g^2*iz`` makes a slab a
  contiguous block, models.cpp:110-112).  Each rank keeps a window of its
  units plus a halo of ``4*K`` units per side and exchanges halos every ``K``
  RK4 steps (deep halos: the 4-stage dependency cone shrinks the valid window
  by 4 units per step).  Every owned unit is computed from exactly the inputs
  a single-device run uses, so the result is bit-identical for any rank count.
* Monte Carlo shards the sample index range; the counter-based RNG needs no
  communication, and the hull is combined with one MIN and one MAX
  all-reduce (exact, order-independent).

The driver is executor-agnostic: ``step_fn`` performs one windowed RK4 step
(on a B200 it is :func:`device_step_fn`, the CUDA kernel through the C ABI)
and ``comm`` moves halo units between neighbours (NCCL point-to-point on
GPUs; the tests drive the same code over gloo).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from .models import HEAT3D, SystemModel


def units_of(model: SystemModel):
    """(number of partition units, components per unit)."""
    if model.kind == HEAT3D:
        return model.grid, model.grid * model.grid
    return model.dim, 1


@dataclass
class Shard:
    """Rank-local partition of ``units`` with a halo of ``halo`` units."""

    units: int
    world: int
    rank: int
    halo: int

    @property
    def begin(self) -> int:
        return self.units * self.rank // self.world

    @property
    def end(self) -> int:
        return self.units * (self.rank + 1) // self.world

    @property
    def win_begin(self) -> int:
        return max(self.begin - self.halo, 0)

    @property
    def win_end(self) -> int:
        return min(self.end + self.halo, self.units)

    @property
    def win_len(self) -> int:
        return self.win_end - self.win_begin

    def out_range(self, s: int):
        """Units computable at sub-step s (0-based) after a halo exchange."""
        shrink = 4 * (s + 1)
        lo = self.win_begin if self.win_begin == 0 else self.win_begin + shrink
        hi = self.win_end if self.win_end == self.units else self.win_end - shrink
        return lo, hi


def plan_rk4_steps(t0: float, t1: float, h: float):
    """(t, hk) per step: rk4.cpp:8-17 and :99-100, in float64 like the host engine."""
    span = t1 - t0
    full = int(np.floor(span / h + 1e-9))
    rem = span - float(full) * h
    total = full + (1 if rem > 1e-9 * h else 0)
    out = []
    for k in range(total):
        t = t0 + float(k) * h
        hk = (t1 - t) if k + 1 == total else h
        out.append((t, hk))
    return out


class HaloExchanger:
    """Sends the rank's boundary units to its neighbours and receives theirs,
    over torch.distributed point-to-point (NCCL on GPUs, gloo in tests)."""

    def __init__(self, shard: Shard, unit: int, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.shard = shard
        self.unit = unit
        self.group = group

    def exchange(self, fields):
        """fields: list of 1-D tensors of length win_len*unit (window layout)."""
        self.finish(self.start(fields))

    def _staged(self) -> bool:
        """gloo cannot move CUDA tensors point-to-point: halos then go through
        host copies (multi-rank tests on one GPU; NCCL moves device memory)."""
        return self.dist.get_backend(self.group) == "gloo"

    def start(self, fields):
        """Post the halo sends / receives and return a handle for finish().  The
        sends read the owned boundary units in place and the receives land
        straight in the window's halo slices (contiguous views: no staging
        buffer, no copy), so the window's owned units may be read meanwhile:
        on GPUs NCCL moves the halos while the interior of the step runs (its
        4-unit stencil cone stays inside the owned units)."""
        s = self.shard
        H = s.halo
        u = self.unit
        ops = []
        staged = []
        left, right = s.rank - 1, s.rank + 1
        wb = s.win_begin
        stage = self._staged()

        def post(snd, rcv, peer):
            if stage and snd.is_cuda:
                snd, dev_rcv = snd.cpu(), rcv
                rcv = dev_rcv.new_empty(dev_rcv.shape, device="cpu")
                staged.append((dev_rcv, rcv))
            ops.append(self.dist.P2POp(self.dist.isend, snd, peer, self.group))
            ops.append(self.dist.P2POp(self.dist.irecv, rcv, peer, self.group))

        for f in fields:
            if left >= 0:
                post(f[(s.begin - wb) * u:(s.begin - wb + H) * u], f[0:(s.begin - wb) * u], left)
            if right < s.world:
                post(f[(s.end - wb - H) * u:(s.end - wb) * u], f[(s.end - wb) * u:(s.win_end - wb) * u], right)
        return (self.dist.batch_isend_irecv(ops) if ops else []), staged

    def finish(self, handle):
        """Wait for the exchange (the halos are already in place, or copied in
        from the host staging buffers on gloo)."""
        reqs, staged = handle
        for r in reqs:
            r.wait()
        for dev, host in staged:
            dev.copy_(host)


class PeerUnavailable(RuntimeError):
    """Neighbouring ranks' GPUs cannot map each other's memory (raised on
    every rank alike by PeerStores.attach)."""


class PeerStores:
    """Halo exchange without a separate transfer, one process per GPU: the
    launch that computes a rank's 4 boundary units stores them a second time,
    over NVLink peer memory, straight into the neighbour's window
    (pirk_step_window_mirror into buffers opened with pirk_ipc_open), then
    raises the neighbour's step flag (pirk_signal_flag); the neighbour's
    stream waits for that flag (pirk_wait_flag, cuStreamWaitValue32) before
    its next boundary launch.  Per step each rank runs
        wait(neighbour flags >= k-1) | boundary units (+ peer stores) |
        signal(k) | interior units
    so a neighbour's next step overlaps this rank's interior.  The flag is
    also the write-after-read guard: the neighbour's halo for step k is in
    the buffer its step k-1 read, and its flag k-1 is raised only after its
    boundary launch (the only reader of the halo) of step k-1.

    ``fused=True`` (default) runs each step as ONE launch over the rank's
    slab that stores its first and last 4 units into the neighbours' windows
    as it computes them:
        wait(neighbour flags >= k-1) | whole slab (+ peer stores) | signal(k)
    A windowed launch pays a fixed cost (the 8-plane z cone and CTA set-up
    over all tiles, ~0.5 ms for heat3d g=1600) however thin it is, so two
    4-unit boundary launches per step cost more than the overlap they buy
    when ranks run in lockstep.  ``fused=False`` keeps the boundary-first
    schedule above.

    Only the control plane (handle exchange, barriers) uses
    torch.distributed, so it runs over NCCL or gloo alike -- on one GPU
    several processes test the same path with device-local "peer" stores.
    Requires K = 1 (halo 4) and every shard at least 8 units wide."""

    def __init__(self, shard: Shard, unit: int, ctx, group=None, fused: bool = True):
        import torch.distributed as dist

        self.dist = dist
        self.shard = shard
        self.unit = unit
        self.ctx = ctx
        self.group = group
        self.fused = fused
        self.seq = 0
        self._bases = []
        if shard.world > 1 and shard.end - shard.begin < 8:
            raise ValueError("peer-store halos need at least 8 units per rank")

    # ---- setup -------------------------------------------------------------
    @staticmethod
    def _export(t):
        import ctypes as C

        from . import _lib

        h = C.create_string_buffer(64)
        off = C.c_uint64(0)
        st = _lib.lib().pirk_ipc_export(C.c_void_p(t.data_ptr()), h, C.byref(off))
        if st != _lib.OK:
            raise RuntimeError(f"pirk_ipc_export failed (status {st})")
        return h.raw, off.value

    def _open(self, device, handle, offset):
        import ctypes as C

        from . import _lib

        base = C.c_void_p(0)
        st = _lib.lib().pirk_ipc_open(int(device), handle, C.byref(base))
        if st != _lib.OK:
            raise RuntimeError(f"pirk_ipc_open failed (status {st})")
        self._bases.append(base.value)
        return base.value + offset

    def attach(self, run: "ShardedReach"):
        """Export this rank's window buffers and flags, map the neighbours'.
        Collective over the group; call after run.alloc().  Raises
        PeerUnavailable on every rank (before mapping anything) when some pair
        of neighbouring GPUs cannot address each other's memory -- the caller
        then uses HaloExchanger."""
        import torch

        s = self.shard
        dev = run.a[0].device
        self.flags = torch.zeros(2, dtype=torch.int32, device=dev)  # [from left, from right]
        self.local = [run.a[0], run.a[1], run.b[0], run.b[1]]
        mine = {"win_begin": s.win_begin, "bufs": [self._export(t) for t in self.local],
                "flags": self._export(self.flags), "device": dev.index,
                "uuid": str(torch.cuda.get_device_properties(dev).uuid)}
        torch.cuda.synchronize(dev)  # flags zeroed before any neighbour can raise them
        allv = [None] * s.world
        self.dist.all_gather_object(allv, mine, group=self.group)
        # every rank checks its own neighbours, then all agree on the outcome
        ok = True
        for r in (s.rank - 1, s.rank + 1):
            if 0 <= r < s.world and allv[r]["uuid"] != mine["uuid"]:
                peer = self._local_index(allv[r]["uuid"])
                ok = ok and peer is not None and torch.cuda.can_device_access_peer(dev.index, peer)
        oks = [None] * s.world
        self.dist.all_gather_object(oks, ok, group=self.group)
        if not all(oks):
            raise PeerUnavailable("peer-store halos need peer access between neighbouring GPUs")
        self.nb = {}
        for side, r in (("left", s.rank - 1), ("right", s.rank + 1)):
            if 0 <= r < s.world:
                o = allv[r]
                self.nb[side] = {"win_begin": o["win_begin"],
                                 "bufs": [self._open(dev.index, *b) for b in o["bufs"]],
                                 "flags": self._open(dev.index, *o["flags"])}
        self.dist.barrier(group=self.group)

    @staticmethod
    def _local_index(uuid: str):
        """This process's index of the device with that UUID (None if not visible)."""
        import torch

        for i in range(torch.cuda.device_count()):
            if str(torch.cuda.get_device_properties(i).uuid) == uuid:
                return i
        return None

    def close(self):
        """Unmap the neighbours' buffers once every rank is done with them."""
        import torch

        from . import _lib

        torch.cuda.synchronize()
        self.dist.barrier(group=self.group)
        for b in self._bases:
            _lib.lib().pirk_ipc_close(b)
        self._bases = []

    # ---- per step ------------------------------------------------------------
    def _on_stream(self, fn, ptr: int, value: int):
        """fn(ctx, ptr, value) on torch's current stream (like device_step_fn)."""
        import torch

        from . import _lib

        prev = _lib.lib().pirk_get_stream(self.ctx.handle)
        self.ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        try:
            self.ctx.check(fn(self.ctx.handle, ptr, value & 0xFFFFFFFF))
        finally:
            self.ctx.set_stream(prev or 0)

    def wait(self, value: int):
        from . import _lib

        for i, side in enumerate(("left", "right")):
            if side in self.nb:
                self._on_stream(_lib.lib().pirk_wait_flag, self.flags.data_ptr() + 4 * i, value)

    def signal(self, value: int):
        from . import _lib

        # I am the right neighbour of my left neighbour: its flags[1]
        for side, slot in (("left", 1), ("right", 0)):
            if side in self.nb:
                self._on_stream(_lib.lib().pirk_signal_flag, self.nb[side]["flags"] + 4 * slot, value)

    def _target(self, side: str, idx: int, out_begin: int):
        """Device address of unit out_begin in the neighbour's buffer idx (the
        address may lie outside that window; only its halo units are stored)."""
        nb = self.nb[side]
        return nb["bufs"][idx] + (out_begin - nb["win_begin"]) * self.unit * 8

    def mirror(self, out0, out_begin: int, out_end: int):
        """pirk_step_window_mirror arguments for a launch over [out_begin,
        out_end): its first 4 units to the left neighbour, its last 4 to the
        right one, into the buffers with the same role (A or B) as this rank's
        out0 -- all ranks swap in lockstep."""
        idx = [t.data_ptr() for t in self.local].index(out0.data_ptr())
        lo = hi = (None, None)
        s = self.shard
        if "left" in self.nb and out_begin < s.begin + 4:
            lo = (self._target("left", idx, out_begin), self._target("left", idx + 1, out_begin))
        if "right" in self.nb and out_end > s.end - 4:
            hi = (self._target("right", idx, out_begin), self._target("right", idx + 1, out_begin))
        return lo[0], lo[1], s.begin + 4, hi[0], hi[1], s.end - 4


def device_step_fn(model: SystemModel, method: str, ctx=None):
    """Windowed RK4 step on the B200 (pirk_step_window on torch tensors), on
    torch's current stream; the context's own stream is restored afterwards."""
    from . import _lib
    from .reach import get_context, step_window

    ctx = ctx or get_context()

    def step(in0, in1, out0, out1, win_begin, win_len, out_begin, out_end, p0, p1, t, hk, k,
             fail_ptr=0, mirror=None):
        import torch

        prev = _lib.lib().pirk_get_stream(ctx.handle)
        ctx.set_stream(torch.cuda.current_stream().cuda_stream)
        try:
            # out pointers address unit out_begin inside the window buffers
            unit = units_of(model)[1]
            off = (out_begin - win_begin) * unit * 8
            step_window(model, method, in0.data_ptr(), in1.data_ptr(), out0.data_ptr() + off,
                        out1.data_ptr() + off, win_begin, win_len, out_begin, out_end, p0, p1, t,
                        hk, k, fail_ptr, ctx=ctx, mirror=mirror)
        finally:
            ctx.set_stream(prev or 0)
    return step


NO_FAIL = (1 << 64) - 1
FAIL_COMP_BITS = 40  # csrc/common.cuh kFailCompBits


def failure_message(method: str, keys, t0: float, h: float):
    """The reference's IntegrationError text (rk4.cpp:19-23 wrapped as in
    reach.cpp:107-117 / :190-192) for the minimum device failure keys
    ``keys`` = (field 0, field 1) -- or None when no step failed."""
    def one(key):
        step, comp = key >> FAIL_COMP_BITS, key & ((1 << FAIL_COMP_BITS) - 1)
        return (f"integration produced a non-finite value at step {step}, component {comp}, "
                f"t = {t0 + float(step) * h:f}")
    if method == "mixed-monotonicity":
        k = min(keys)
        return None if k == NO_FAIL else "mixed-monotonicity embedding integration: " + one(k)
    if keys[0] != NO_FAIL:
        return "growth-bound center integration: " + one(keys[0])
    if keys[1] != NO_FAIL:
        return "growth-bound radius integration: " + one(keys[1])
    return None


class ShardedReach:
    """Runs the RK4 step loop of one shard: window buffers (two fields,
    ping-pong), ``K``-step deep halos.  Tensors may live on any torch device
    the ``step_fn`` understands."""

    def __init__(self, model: SystemModel, method: str, shard: Shard, step_fn: Callable,
                 exchanger: Optional[HaloExchanger], p0=None, p1=None, K: int = 1):
        assert shard.halo == 4 * K, "halo must be 4*K units for K steps between exchanges"
        self.model = model
        self.method = method
        self.shard = shard
        self.step_fn = step_fn
        self.ex = exchanger
        self.p0, self.p1 = p0, p1
        self.K = K
        self.unit = units_of(model)[1]

    def alloc(self, like_tensor_factory, fail=None):
        """Window buffers from ``like_tensor_factory(n)``; ``fail`` is an
        optional device tensor of two uint64 failure keys (all ones = none)
        that every step's kernels atomically lower (see check())."""
        n = self.shard.win_len * self.unit
        self.a = [like_tensor_factory(n), like_tensor_factory(n)]
        self.b = [like_tensor_factory(n), like_tensor_factory(n)]
        self.fail = fail
        return self.a

    def _fail_ptr(self):
        f = getattr(self, "fail", None)
        return 0 if f is None else f.data_ptr()

    def check(self, t0: float, h: float, group=None):
        """Raise the reference's IntegrationError (as RuntimeError) if any rank's
        kernels saw a non-finite value: the per-rank minimum keys are combined
        with a MIN all-reduce, so every rank raises the same message."""
        f = getattr(self, "fail", None)
        if f is None:
            return
        import torch

        v = f.view(torch.int64).clone()
        big = torch.iinfo(torch.int64).max
        v = torch.where(v == -1, torch.full_like(v, big), v)  # no failure -> +inf
        import torch.distributed as dist
        if self.shard.world > 1 and dist.is_available() and dist.is_initialized():
            if dist.get_backend(group) == "gloo":
                v = v.cpu()
            dist.all_reduce(v, op=dist.ReduceOp.MIN, group=group)
        keys = [NO_FAIL if int(x) == big else int(x) for x in v.cpu().tolist()]
        msg = failure_message(self.method, keys, t0, h)
        if msg:
            raise RuntimeError(msg)

    def run(self, steps, k0: int = 0, overlap: bool = True):
        """steps: list of (t, hk) for global step indices k0, k0+1, ...

        On an exchange step with ``overlap`` the halos move while the units
        whose stencil cone (4 units per RK4 step) lies inside the rank's own
        units are computed; the units next to the window edges follow once
        the halos have landed.  Every unit is still computed once, from the
        same inputs, so results do not depend on ``overlap``."""
        if isinstance(self.ex, PeerStores):
            return self._run_peer(steps, k0)
        s = self.shard
        fp = self._fail_ptr()
        for i, (t, hk) in enumerate(steps):
            sub = (k0 + i) % self.K
            lo, hi = s.out_range(sub)
            args = (s.win_begin, s.win_len)
            if sub == 0 and self.ex is not None and s.world > 1:
                if overlap:
                    handle = self.ex.start(self.a)
                    ilo, ihi = max(lo, s.begin + 4), min(hi, s.end - 4)
                    if ilo < ihi:  # interior: independent of the incoming halos
                        self.step_fn(self.a[0], self.a[1], self.b[0], self.b[1], *args, ilo, ihi,
                                     self.p0, self.p1, t, hk, k0 + i, fp)
                    self.ex.finish(handle)
                    for blo, bhi in ((lo, min(hi, ilo)), (max(lo, ihi), hi)) if ilo < ihi else ((lo, hi),):
                        if blo < bhi:
                            self.step_fn(self.a[0], self.a[1], self.b[0], self.b[1], *args, blo, bhi,
                                         self.p0, self.p1, t, hk, k0 + i, fp)
                    self.a, self.b = self.b, self.a
                    continue
                self.ex.exchange(self.a)
            self.step_fn(self.a[0], self.a[1], self.b[0], self.b[1], *args, lo, hi, self.p0, self.p1, t,
                         hk, k0 + i, fp)
            self.a, self.b = self.b, self.a

    def _run_peer(self, steps, k0: int):
        """Boundary units first, stored into the neighbours' windows by the
        same launch; then the interior (see PeerStores)."""
        s, ex = self.shard, self.ex
        assert self.K == 1, "peer-store halos exchange every step (K = 1)"
        fp = self._fail_ptr()
        args = (s.win_begin, s.win_len)
        has_l, has_r = "left" in ex.nb, "right" in ex.nb
        ilo = s.begin + 4 if has_l else s.begin
        ihi = s.end - 4 if has_r else s.end
        for i, (t, hk) in enumerate(steps):
            ex.seq += 1
            ex.wait(ex.seq - 1)
            a, b = self.a, self.b
            if ex.fused:
                mir = ex.mirror(b[0], s.begin, s.end) if ex.nb else None
                self.step_fn(a[0], a[1], b[0], b[1], *args, s.begin, s.end, self.p0, self.p1, t, hk, k0 + i,
                             fp, mirror=mir)
                ex.signal(ex.seq)
            else:
                for side, (blo, bhi) in (("left", (s.begin, s.begin + 4)), ("right", (s.end - 4, s.end))):
                    if side in ex.nb:
                        self.step_fn(a[0], a[1], b[0], b[1], *args, blo, bhi, self.p0, self.p1, t, hk, k0 + i,
                                     fp, mirror=ex.mirror(b[0], blo, bhi))
                ex.signal(ex.seq)
                if ilo < ihi:
                    self.step_fn(a[0], a[1], b[0], b[1], *args, ilo, ihi, self.p0, self.p1, t, hk, k0 + i, fp)
            self.a, self.b = b, a

    def owned(self):
        s = self.shard
        u = self.unit
        o0 = (s.begin - s.win_begin) * u
        o1 = (s.end - s.win_begin) * u
        return self.a[0][o0:o1], self.a[1][o0:o1]


def mc_sample_range(m: int, world: int, rank: int):
    return m * rank // world, m * (rank + 1) // world


def allreduce_hull(lower, upper, group=None):
    """Combine per-rank Monte Carlo hulls (torch tensors): exact MIN/MAX."""
    import torch.distributed as dist

    dist.all_reduce(lower, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(upper, op=dist.ReduceOp.MAX, group=group)
