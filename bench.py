"""Benchmark of the PIRK reachability hot path on B200.

Default workload (BASELINE.json config 5 / north-star target): CTMM
(mixed monotonicity) of heat3d with grid = 1600 (n = 4.096e9, embedding state
2n = 8.19e9 fp64), h = 5e-8, strong-scaled over N GPUs as z-slabs whose
boundary launches store their halo planes straight into the neighbours'
windows over NVLink (--halo peer; --halo nccl: NCCL send/recv).  One bench "step" is one RK4 step of the whole embedding.

* value  -- state-updates/s (2n per step) with the state resident in HBM,
            CUDA events on the launching stream, max over ranks.
* e2e    -- the same metric through the public API (paper_2001_10635_b200.
            mixed_monotonicity, host buffers in and out, H2D/D2H in the timed
            region) for the full 100-step C5 reach.
* roofline, cpu_baseline (the reference itself, oracle/_ref, on this host),
  clocks, gpu_launches -- see DESIGN.md.

``--impl reference`` times the reference's own CPU implementation (oracle/_ref,
built from /root/reference/proj/src) on bounded samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RK4 state-updates/sec (2n*steps/s), CTMM heat3d n=4.096e9"
UNIT = "state-updates/s"
GRID = 1600
H = 5e-8
C5_STEPS = 100


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def heat_kernel_name(mode, grid):
    """The heat kernel launch_heat_step (csrc/heat2x2.cuh) runs for this mode and
    grid: warp-wide strips in fast mode (TMA path: even g), 1x2 pairs in exact
    mode; PIRK_HEAT_BLOCK=1x2|2x2|4x4|strip overrides."""
    v = os.environ.get("PIRK_HEAT_BLOCK", "")
    if mode == "fast" and grid % 2 == 0 and v in ("", "strip", "4x4"):
        return "heat4_step_kernel" if v == "4x4" else "heat_strip_kernel"
    if v == "1x2" or (v == "" and mode != "fast"):
        return "heat_step_kernel"
    return "heat2_step_kernel"


def allreduce(dist, t, op):
    """All-reduce a device tensor in place (through the host on gloo, which
    the one-GPU multi-rank test of the N > 1 path uses)."""
    if dist.get_backend() == "gloo":
        c = t.cpu()
        dist.all_reduce(c, op=op)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=op)


def device_of(args, local):
    """cuda device of a rank: its LOCAL_RANK, or 0 for --same-device (testing
    the N > 1 code path with several ranks on one GPU)."""
    return 0 if args.same_device else local


def halo_exchanger(args, S, shard, unit, ctx, world):
    """N > 1 halo transport of the heat runs: peer stores fused into the
    boundary launches (--halo peer, default: CUDA IPC over NVLink, no
    separate transfer) or NCCL send/recv (--halo nccl)."""
    if world == 1:
        return None
    if args.halo == "peer":
        return S.PeerStores(shard, unit, ctx)
    return S.HaloExchanger(shard, unit)


def attach_or_nccl(args, S, run, ex, shard, unit):
    """Map the neighbours' windows for peer stores; if some neighbouring GPUs
    cannot address each other (every rank learns it together), the run uses
    NCCL halo exchange instead and the line says so (args.halo)."""
    if not isinstance(ex, S.PeerStores):
        return ex
    try:
        ex.attach(run)
        return ex
    except S.PeerUnavailable:
        args.halo = "nccl"
        run.ex = S.HaloExchanger(shard, unit)
        return run.ex


HALO_DESC = {"peer": "halos stored into the neighbours' windows by the boundary launches (CUDA IPC peer memory)",
             "nccl": "NCCL halo exchange"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------- our arm

def heat_device_bench(args, world, rank, local, torch, pk, dist):
    """Device-resident CTMM steps of heat3d (sharded z-slabs for N > 1)."""
    from paper_2001_10635_b200 import sharded as S

    model = pk.make_heat3d(args.grid)
    local = device_of(args, local)
    ctx = pk.Context(local, args.mode)
    K = 1
    shard = S.Shard(args.grid, world, rank, 4 * K)
    unit = args.grid * args.grid
    ex = halo_exchanger(args, S, shard, unit, ctx, world)
    step_fn = S.device_step_fn(model, "mixed-monotonicity", ctx)
    run = S.ShardedReach(model, "mixed-monotonicity", shard, step_fn, ex, K=K)
    dev = torch.device("cuda", local)
    fail = torch.full((2,), -1, dtype=torch.int64, device=dev)  # device failure keys
    a = run.alloc(lambda n: torch.empty(n, dtype=torch.float64, device=dev), fail=fail)
    ex = attach_or_nccl(args, S, run, ex, shard, unit)
    a[0].fill_(0.9)  # catalog default box [0.9, 1.1] (models.cpp:744-745)
    a[1].fill_(1.1)
    steps = [(float(k) * args.h, args.h) for k in range(args.warmup + args.steps)]
    launches0 = ctx.launch_count()
    torch.cuda.synchronize()
    stream = torch.cuda.Stream(device=dev)  # kernels and events share this stream
    with torch.cuda.stream(stream):
        run.run(steps[: args.warmup], 0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        l0 = ctx.launch_count()
        with torch.cuda.stream(stream):
            ev0.record(stream)
            run.run(steps[args.warmup:], args.warmup)
            ev1.record(stream)
        torch.cuda.synchronize()
        l1 = ctx.launch_count()
        if world > 1:
            dist.barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        allreduce(dist, t, dist.ReduceOp.MAX)
    ms_max = float(t.item())
    run.check(0.0, args.h)  # raises the reference's IntegrationError on any rank's failure
    check = state_check(run, args, torch, dist, world)
    if isinstance(ex, S.PeerStores):
        ex.close()
    del a, run
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    ctx.close()
    return ms_max, l1 - l0, clk.summary(), check, launches0


def state_check(run, args, torch, dist, world):
    """Checks of the device result after the timed steps, on every rank's owned
    slab (cheap device reductions, no copy back):
      * finite, lower <= upper, and within [0, 1.1] (the maximum principle of
        a diffusion with Robin loss from the box [0.9, 1.1]);
      * plane invariance: from the catalog's uniform box the heat field is
        constant on every (y, z) plane (only the x = 0 face exchanges heat,
        models.cpp:116-125), so every row of g components must equal the
        first row -- bit-exact in exact mode, <= 1e-12 relative in fast mode.
        tests/test_gpu_scale.py checks the same rows against the reference
        arithmetic at this full size."""
    lo, hi = run.owned()
    g = args.grid
    r0_lo = lo[:g].clone()
    r0_hi = hi[:g].clone()
    worst = torch.zeros((), dtype=torch.float64, device=lo.device)
    ok = torch.ones((), dtype=torch.bool, device=lo.device)
    rows_lo, rows_hi = lo.view(-1, g), hi.view(-1, g)
    for c0 in range(0, rows_lo.shape[0], 1 << 18):
        bl, bh = rows_lo[c0:c0 + (1 << 18)], rows_hi[c0:c0 + (1 << 18)]
        ok &= torch.isfinite(bl).all() & torch.isfinite(bh).all() & (bl <= bh).all()
        ok &= (bl >= 0).all() & (bh <= 1.1).all()
        worst = torch.maximum(worst, ((bl - r0_lo).abs() / r0_lo.abs()).max())
        worst = torch.maximum(worst, ((bh - r0_hi).abs() / r0_hi.abs()).max())
    # the first row of every rank is the same physical line: compare rank 0's
    v = torch.stack([ok.to(torch.float64), -worst])
    if world > 1:
        allreduce(dist, v, dist.ReduceOp.MIN)
    return {"finite_ordered_bounded": bool(v[0].item() == 1.0),
            "plane_invariance_max_rel": float(-v[1].item()),
            "plane_invariance_ok": float(-v[1].item()) <= (0.0 if args.mode == "exact" else 1e-12)}


def heat_e2e(args, pk, torch, world):
    """Full C5 reach (100 steps, final set) through the public API with host
    buffers; H2D of the initial box and D2H of the final box are timed."""
    import psutil

    g = args.grid
    n = g ** 3
    need = 4 * n * 8
    avail = psutil.virtual_memory().available
    if need > 0.75 * avail:
        # keep the box alive: scale the e2e grid down rather than exhaust host RAM
        g = int(round((0.75 * avail / 32) ** (1.0 / 3.0)))
        n = g ** 3
    # page-locked host buffers via cudaHostRegister (torch's pinned allocator
    # rounds requests up to powers of two, which would not fit host RAM here)
    bufs = [np.empty(n) for _ in range(4)]
    cudart = torch.cuda.cudart()
    for b in bufs:
        cudart.cudaHostRegister(b.ctypes.data, b.nbytes, 0)
    lo, hi, olo, ohi = bufs
    lo.fill(0.9)
    hi.fill(1.1)
    model = pk.make_heat3d(g)
    # IntervalVector validation is part of problem construction (interval.cpp:10-23),
    # outside the reference's mixed_monotonicity call; done before timing here too.
    prob = pk.ReachProblem(model, pk.IntervalVector(lo, hi), None, 0.0,
                           C5_STEPS * args.h, args.h, 0)
    ctx = pk.get_context(0)
    ctx.set_mode(args.mode)
    # one untimed call first: the driver maps freshly registered host pages on
    # their first DMA (the first upload of each 32 GB buffer runs synchronously),
    # which is setup like the registration itself, not per-call work.  It also
    # leaves the 4 state buffers in the context's cache (engine.cu), so the
    # next call is the steady-state ("warm") one; after release_cache() the
    # call pays the 131 GB of cudaMalloc again ("cold").
    pk.mixed_monotonicity(prob, ctx=ctx, out=(olo, ohi))
    t0 = time.perf_counter()
    tube = pk.mixed_monotonicity(prob, ctx=ctx, out=(olo, ohi))
    dt = time.perf_counter() - t0
    ok = bool(np.isfinite(olo[:: max(1, n // 4096)]).all())
    ctx.release_cache()
    t1 = time.perf_counter()
    cold = pk.mixed_monotonicity(prob, ctx=ctx, out=(olo, ohi))
    dt_cold = time.perf_counter() - t1
    ctx.release_cache()
    steps = tube.report.steps
    res = {"value": 2.0 * n * steps / dt, "unit": UNIT, "h2d_bytes_per_step": 2 * n * 8,
           "d2h_bytes_per_step": 2 * n * 8, "seconds": dt, "rk4_steps": steps,
           "n": n, "grid": g, "api": "paper_2001_10635_b200.mixed_monotonicity",
           "step": "one full C5 reach call (H2D initial box, 100 RK4 steps, order check, D2H final box); "
                   "lower field integrated while the upper field uploads, downloaded while it integrates; "
                   "skewed rounds start the lower field on its first uploaded planes and send the upper "
                   "field's final planes back in strips (engine.cu skew_fronts)",
           "warmup_calls": 1, "state_cache": "warm (the 4 state buffers kept by the previous call)",
           "cold": {"value": 2.0 * n * cold.report.steps / dt_cold, "seconds": dt_cold,
                    "state_cache": "cold (release_cache() before the call: cudaMalloc of the state inside)"},
           "phases_s": {"setup": tube.report.phases.setup_s,
                        "integration_incl_transfers": tube.report.phases.integration_s}}
    del tube, cold, prob, lo, hi, olo, ohi
    for b in bufs:
        cudart.cudaHostUnregister(b.ctypes.data)
    del bufs
    return res, ok


def heat_e2e_sharded(args, pk, torch, dist, world, rank, local):
    """N > 1 end to end: the full C5 reach (100 steps) through the sharded
    public API with host buffers per rank.  Each rank uploads its window of the
    initial box from page-locked host memory, integrates with the --halo
    transport (peer stores or NCCL), checks the embedding order on its slab and downloads its slab of
    the final box; time = max over ranks of the whole call."""
    from paper_2001_10635_b200 import sharded as S

    g = args.grid
    unit = g * g
    model = pk.make_heat3d(g)
    local = device_of(args, local)
    ctx = pk.Context(local, args.mode)
    shard = S.Shard(g, world, rank, 4)
    dev = torch.device("cuda", local)
    win, own = shard.win_len * unit, (shard.end - shard.begin) * unit
    # page-locked through cudaHostRegister (torch's pinned allocator rounds up to
    # powers of two: 8 ranks x 4 x 8 GB would not fit a host)
    host = [np.empty(win), np.empty(win), np.empty(own), np.empty(own)]
    cudart = torch.cuda.cudart()
    for b in host:
        cudart.cudaHostRegister(b.ctypes.data, b.nbytes, 0)
    host[0].fill(0.9)
    host[1].fill(1.1)
    h_lo, h_hi, o_lo, o_hi = (torch.from_numpy(b) for b in host)
    ex = halo_exchanger(args, S, shard, unit, ctx, world)
    run = S.ShardedReach(model, "mixed-monotonicity", shard, S.device_step_fn(model, "mixed-monotonicity", ctx),
                         ex, K=1)
    steps = S.plan_rk4_steps(0.0, C5_STEPS * args.h, args.h)
    fail = torch.full((2,), -1, dtype=torch.int64, device=dev)
    a = run.alloc(lambda k: torch.empty(k, dtype=torch.float64, device=dev), fail=fail)
    ex = attach_or_nccl(args, S, run, ex, shard, unit)
    stream = torch.cuda.Stream(device=dev)

    def once():
        with torch.cuda.stream(stream):
            fail.fill_(-1)
            run.a[0].copy_(h_lo, non_blocking=True)
            run.a[1].copy_(h_hi, non_blocking=True)
            run.run(steps, 0)
            lo, hi = run.owned()
            bad = (lo > hi).any()  # reach.cpp:181-186 on this slab
            o_lo.copy_(lo, non_blocking=True)
            o_hi.copy_(hi, non_blocking=True)
        stream.synchronize()
        run.check(0.0, args.h)
        return bool(bad.item())

    once()  # warm-up call (NCCL connections, page-locked mappings)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    bad = once()
    dt = time.perf_counter() - t0
    tt = torch.tensor([dt, float(bad)], dtype=torch.float64, device=dev)
    allreduce(dist, tt, dist.ReduceOp.MAX)
    n = g ** 3
    res = {"value": 2.0 * n * len(steps) / tt[0].item(), "unit": UNIT,
           "h2d_bytes_per_step": 2 * 8 * (n + 2 * (world - 1) * 4 * unit), "d2h_bytes_per_step": 2 * n * 8,
           "seconds": tt[0].item(), "rk4_steps": len(steps), "n": n, "grid": g,
           "api": f"paper_2001_10635_b200.sharded.ShardedReach (one process per GPU, {HALO_DESC[args.halo]})",
           "order_violated": bool(tt[1].item()), "timing": "wall clock of the whole call, max over ranks"}
    if isinstance(ex, S.PeerStores):
        ex.close()
    del a, run, h_lo, h_hi, o_lo, o_hi
    for b in host:
        cudart.cudaHostUnregister(b.ctypes.data)
    torch.cuda.empty_cache()
    ctx.close()
    return res


def fp64_peak():
    """Measured FP64 pipe peak (profiles/r02_fp64_peak.json, DFMA/DADD/DMUL
    microbenchmark on this pool's B200): instructions/s (the largest of the
    three, so fractions are conservative) and TFLOP/s (DFMA = 2 flops)."""
    with open(os.path.join(ROOT, "profiles", "r02_fp64_peak.json")) as f:
        p = json.load(f)
    return max(p["dfma_per_s"], p["dadd_per_s"], p["dmul_per_s"]), p["fp64_tflops_fma"]


def fp64_counts():
    """Executed FP64 instructions / flops per unit of work of each secondary
    kernel (ncu SASS counters, profiles/r02_fp64_counts.json)."""
    with open(os.path.join(ROOT, "profiles", "r02_fp64_counts.json")) as f:
        return json.load(f)["kernels"]


def fp64_roofline(rate, key, kernel):
    inst_peak, tflops_peak = fp64_peak()
    c = fp64_counts()[key]
    inst = c["fp64_inst_per_unit"] * rate
    flops = c["fp64_flops_per_unit"] * rate
    return {"bound": "fp64", "achieved": inst / 1e12, "peak": inst_peak / 1e12,
            "unit": "T FP64 inst/s", "frac": inst / inst_peak,
            "achieved_tflops": flops / 1e12, "peak_tflops": tflops_peak,
            "frac_flops": flops / 1e12 / tflops_peak, "kernel": kernel,
            "fp64_inst_per_unit": c["fp64_inst_per_unit"], "fp64_flops_per_unit": c["fp64_flops_per_unit"],
            "ncu_pipe_fp64_pct": c["pipe_fp64_pct"],
            "counts_from": "profiles/r02_fp64_counts.json (ncu SASS counters); peak: profiles/r02_fp64_peak.json"}


def host_ram_gb():
    import psutil

    vm = psutil.virtual_memory()
    return vm.total / 2 ** 30, vm.available / 2 ** 30


def host_cpu():
    """CPU model and logical CPU count of this host (report them
    beside the reference timing)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def cpu_baseline(args):
    """The reference itself (oracle/_ref) on this host, bounded sample at the
    largest heat3d grid the host RAM holds (the reference keeps 7 vectors of
    2n doubles, 112n bytes, plus the 4n-double box arrays here), capped so the
    sample is ~20 s of CPU work (C5's g = 1600 needs 459 GB)."""
    from oracle import oracle as O

    import paper_2001_10635_b200 as pk

    if not O.ref_available():
        return None
    total_gb, avail_gb = host_ram_gb()
    g_ram = int((0.8 * avail_gb * 2 ** 30 / 150.0) ** (1.0 / 3.0))
    g = max(args.cpu_grid, min(g_ram, args.cpu_grid_max))
    steps = args.cpu_steps
    model = pk.make_heat3d(g)
    n = g ** 3
    threads = O.ref_max_threads()
    r = O.ref_reach(O.METHOD_MM, model, np.full(n, 0.9), np.full(n, 1.1), None, None, 0.0,
                    steps * args.h, args.h, 0, workers=threads, keep=False)
    rate = 2.0 * n * steps / r.report["integration_s"]
    # the same reference on one worker (all cores and 1), on a
    # small grid to stay within the bench's time budget
    g1, s1 = 300, 2
    n1 = g1 ** 3
    r1 = O.ref_reach(O.METHOD_MM, pk.make_heat3d(g1), np.full(n1, 0.9), np.full(n1, 1.1), None, None,
                     0.0, s1 * args.h, args.h, 0, workers=1, keep=False)
    return {"value": rate, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"ivreach::mixed_monotonicity (oracle/_ref, -O3, OpenMP, x86-64 baseline, no FMA) "
                      f"heat3d grid={g} (n={n}), {steps} RK4 steps, h={args.h}; rate = 2n*steps/integration_s; "
                      f"grid = the largest the host RAM holds (capped at {args.cpu_grid_max})",
            **host_cpu(),
            "host_ram_gb": round(total_gb, 1), "host_ram_available_gb": round(avail_gb, 1),
            "reference_state_gb": round(112.0 * n / 1e9, 1),
            "wall_s": r.wall_s, "integration_s": r.report["integration_s"],
            "single_worker": {"value": 2.0 * n1 * s1 / r1.report["integration_s"], "cores": 1,
                              "grid": g1, "steps": s1}}


def secondary(args, pk, torch):
    """The other BASELINE configs on one GPU, each with the roofline that
    bounds it and the reference timed beside it on the host cores."""
    from oracle import oracle as O

    out = {}
    ctx = pk.get_context(0)
    ctx.set_mode(args.mode)
    ref_ok = O.ref_available() and not args.no_cpu
    threads = O.ref_max_threads() if ref_ok else 0

    def engine_rate(prob, steps=20):
        eng = pk.Engine(prob, ctx=ctx)
        stream = torch.cuda.Stream()
        ctx.set_stream(stream.cuda_stream)
        eng.advance(3)
        eng.status()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.advance(steps)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / steps
        eng.close()
        ctx.set_stream(None)
        return 2.0 * prob.model.dim / (ms * 1e-3), ms

    def ref_rate(method, prob, **kw):
        p = prob
        plo = p.inputs.lower if p.inputs is not None else None
        phi = p.inputs.upper if p.inputs is not None else None
        r = O.ref_reach(method, p.model, p.initial.lower, p.initial.upper, plo, phi, p.t0, p.t1, p.h,
                        p.tube_stride, workers=threads, keep=False, **kw)
        return r

    hbm, _ = peaks()
    # C3: traffic n = 1e6 CTMM.  The 4 state buffers (32 MB) stay in the 126 MB
    # L2 and a step is ~10 us: launch / latency and the FP64 pipe bound it, not
    # HBM (the HBM fraction is kept for comparison only).
    n = 10 ** 6
    m = pk.make_traffic(n)
    p = pk.ReachProblem(m, pk.IntervalVector(np.full(n, 10.0), np.full(n, 20.0)),
                        pk.IntervalVector([4.0], [6.0]), 0.0, 30.0, 0.5, 0)
    v, ms = engine_rate(p, 40)
    c3 = {"value": v, "unit": UNIT, "ms_per_step": ms, "kernel": "chain_warp_kernel",
          "roofline": fp64_roofline(v, f"traffic_{args.mode}", "chain_warp_kernel"),
          "hbm_frac_if_streamed": v * 16.0 / (hbm * 1e9),
          "note": "state (4 x 8 MB) is L2-resident; ~10 us per RK4 step"}
    if ref_ok:
        r = ref_rate(O.METHOD_MM, p)
        c3["cpu_baseline"] = {"value": 2.0 * n * r.report["steps"] / r.report["integration_s"], "unit": UNIT,
                              "cores": threads, "kind": "reference",
                              "sample": "ivreach::mixed_monotonicity traffic n=1e6, 60 steps (the full C3 reach)"}
    out["C3_traffic_ctmm_n1e6"] = c3
    # C4: coupled chain n = 1e7 (SDMM interpretation): FP64-bound
    n = 10 ** 7
    m = pk.make_chain(n)
    ctr = 2.0 * O.u01_vec(7, 0, np.arange(n, dtype=np.uint64)) - 1.0
    p = pk.ReachProblem(m, pk.IntervalVector(ctr - 0.05, ctr + 0.05), pk.IntervalVector([-0.1], [0.1]),
                        0.0, 1.0, 0.01, 0)
    v, ms = engine_rate(p, 40)
    c4 = {"value": v, "unit": UNIT, "ms_per_step": ms, "kernel": "chain_warp_kernel",
          "roofline": fp64_roofline(v, f"chain_{args.mode}", "chain_warp_kernel"),
          "hbm_frac": v * 16.0 / (hbm * 1e9)}
    if ref_ok:
        p10 = pk.ReachProblem(m, p.initial, p.inputs, 0.0, 0.1, 0.01, 0)
        r = ref_rate(O.METHOD_MM, p10)
        c4["cpu_baseline"] = {"value": 2.0 * n * r.report["steps"] / r.report["integration_s"], "unit": UNIT,
                              "cores": threads, "kind": "reference",
                              "sample": "ivreach::mixed_monotonicity chain n=1e7, first 10 of the 100 steps"}
    out["C4_chain_sdmm_n1e7"] = c4
    # C1: CTMM of the 12-state arch-quadrotor (Jacobian-bound decomposition,
    # SURVEY.md 8d), 100 steps, stride 10: one small embedding integrated by one
    # device thread -- latency-bound; reported with the reference beside it
    mq = pk.with_jacobian_decomposition(pk.make_arch_quadrotor())
    lo = np.array([-0.4] * 6 + [0.0] * 6)
    p = pk.ReachProblem(mq, pk.IntervalVector(lo, -lo), None, 0.0, 1.0, 0.01, 10)
    pk.mixed_monotonicity(p, ctx=ctx)
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        tube = pk.mixed_monotonicity(p, ctx=ctx)
    dt = (time.perf_counter() - t0) / reps
    c1 = {"value": 24.0 * tube.report.steps / dt, "unit": UNIT, "call_ms": dt * 1e3,
          "kernel_ms": tube.report.phases.integration_s * 1e3,
          "bound": "latency: one device thread integrates the 24-dimensional embedding (RK4 stages are "
                   "sequential); a single small problem does not fill a GPU"}
    if ref_ok:
        r1 = O.ref_reach(O.METHOD_MM, mq, lo, -lo, None, None, 0.0, 1.0, 0.01, 10, workers=1, keep=False)
        c1["cpu_baseline"] = {"value": 24.0 * r1.report["steps"] / r1.report["integration_s"], "unit": UNIT,
                              "cores": 1, "kind": "reference",
                              "sample": "ivreach::mixed_monotonicity arch-quadrotor (Jacobian decomposition), "
                                        "the full C1 reach on one worker"}
    out["C1_archquad_ctmm_n12"] = c1
    # C2: arch-quadrotor Monte Carlo, m = 1e6, 100 steps: FP64-bound
    mq = pk.make_arch_quadrotor()
    lo = np.array([-0.4] * 6 + [0.0] * 6)
    p = pk.ReachProblem(mq, pk.IntervalVector(lo, -lo), None, 0.0, 1.0, 0.01, 0)
    spec = pk.MonteCarloSpec(seed=1, samples_override=10 ** 6)
    pk.monte_carlo(p, pk.MonteCarloSpec(seed=1, samples_override=10 ** 5), ctx=ctx)
    t0 = time.perf_counter()
    tube = pk.monte_carlo(p, spec, ctx=ctx)
    dt = time.perf_counter() - t0
    kv = 1e6 * tube.report.steps / tube.report.phases.integration_s
    c2 = {"value": 1e6 * tube.report.steps / dt, "unit": "sample-steps/s",
          "kernel_s": tube.report.phases.integration_s, "kernel_value": kv,
          "roofline": fp64_roofline(kv, f"mc_{args.mode}", "monte_carlo_kernel")}
    if ref_ok:
        ms_ = 10 ** 5
        r = ref_rate(O.METHOD_MC, p, samples=ms_, seed=1)
        c2["cpu_baseline"] = {"value": ms_ * r.report["steps"] / r.report["integration_s"],
                              "unit": "sample-steps/s", "cores": threads, "kind": "reference",
                              "sample": f"ivreach::monte_carlo arch-quadrotor m={ms_} (of 1e6), 100 steps"}
    out["C2_archquad_mc_m1e6"] = c2
    return out


def sharded_chain_bench(args, world, rank, local, torch, pk, dist):
    """BASELINE config 4 at N GPUs: the coupled chain n = 1e7 sharded into
    index ranges with deep halos (K = 8 steps per exchange, 32-unit halos: the
    1-D halo is pure latency), NCCL point-to-point between ranks; 100-step
    reach timed on the device, max over ranks."""
    from paper_2001_10635_b200 import sharded as S

    n, K, steps = args.chain_n, 8, 100
    model = pk.make_chain(n)
    local = device_of(args, local)
    ctx = pk.Context(local, args.mode)
    shard = S.Shard(n, world, rank, 4 * K)
    run = S.ShardedReach(model, "mixed-monotonicity", shard, S.device_step_fn(model, "mixed-monotonicity", ctx),
                         S.HaloExchanger(shard, 1) if world > 1 else None, [-0.1], [0.1], K=K)
    dev = torch.device("cuda", local)
    fail = torch.full((2,), -1, dtype=torch.int64, device=dev)
    a = run.alloc(lambda k: torch.empty(k, dtype=torch.float64, device=dev), fail=fail)
    idx = torch.arange(shard.win_begin, shard.win_end, dtype=torch.float64, device=dev)
    a[0].copy_(torch.sin(idx) - 0.05)
    a[1].copy_(torch.sin(idx) + 0.05)
    plan = S.plan_rk4_steps(0.0, steps * 0.01, 0.01)
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        run.run(plan[:K], 0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        run.run(plan[K:], K)
        e1.record(stream)
    torch.cuda.synchronize()
    run.check(0.0, 0.01)
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        allreduce(dist, t, dist.ReduceOp.MAX)
    ms = float(t.item())
    del a, run
    torch.cuda.empty_cache()
    ctx.close()
    timed = steps - K
    return {"value": 2.0 * n * timed / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms / timed,
            "n_gpus": world, "halo_units": 4 * K, "steps_per_exchange": K,
            "workload": f"C4 coupled chain n={n} CTMM, index-range shards, {dist.get_backend() if world > 1 else 'no'} halos, "
                        f"{timed} timed steps",
            "scaling": "strong"}


def sharded_mc_bench(args, world, rank, local, torch, pk, dist):
    """BASELINE config 2 at N GPUs: arch-quadrotor Monte Carlo, m = 1e6 samples
    split into per-rank index ranges (counter-based draws: no communication),
    each rank folding its hull (pirk_monte_carlo_range), then one MIN and one
    MAX all-reduce of the hull; wall time of the whole call
    including the reduction, max over ranks."""
    from paper_2001_10635_b200 import sharded as S

    local = device_of(args, local)
    ctx = pk.Context(local, args.mode)
    mq = pk.make_arch_quadrotor()
    lo = np.array([-0.4] * 6 + [0.0] * 6)
    prob = pk.ReachProblem(mq, pk.IntervalVector(lo, -lo), None, 0.0, 1.0, 0.01, 0)
    m = 10 ** 6
    b, e = S.mc_sample_range(m, world, rank)

    def once():
        flo = np.full((1, 12), np.inf)
        fhi = np.full((1, 12), -np.inf)
        pk.monte_carlo_range(prob, 1, b, e, flo, fhi, ctx=ctx)
        if world > 1:
            tl, th = torch.from_numpy(flo), torch.from_numpy(fhi)
            if dist.get_backend() != "gloo":
                tl, th = tl.cuda(local), th.cuda(local)
            S.allreduce_hull(tl, th)
            flo, fhi = tl.cpu().numpy(), th.cpu().numpy()
        return flo, fhi

    once()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    flo, fhi = once()
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64, device=torch.device("cuda", local))
    if world > 1:
        allreduce(dist, t, dist.ReduceOp.MAX)
    ctx.close()
    ok = bool(np.isfinite(flo).all() and np.isfinite(fhi).all() and (flo <= fhi).all())
    return {"value": m * 100 / float(t.item()), "unit": "sample-steps/s", "seconds": float(t.item()),
            "n_gpus": world, "samples": m, "hull_ok": ok, "scaling": "strong",
            "workload": "C2 arch-quadrotor MC m=1e6, 100 steps, sample ranges per rank + MIN/MAX all-reduce"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2001_10635_b200 as pk

    world, rank, local = dist_env()
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", device_of(args, local)))
        else:
            dist.init_process_group("gloo")
    torch.cuda.set_device(device_of(args, local))
    pk.set_default_mode(args.mode)
    ms, launches, clocks, check, _ = heat_device_bench(args, world, rank, local, torch, pk, dist)
    n = args.grid ** 3
    updates = 2.0 * n * args.steps
    value = updates / (ms * 1e-3)
    hbm, how = peaks()
    # dominant kernel: the heat step kernel.  At N = 1 it is one launch per
    # step; at N > 1 a step is 1-3 launches of it (interior + boundary slabs)
    # and the roofline is taken per step: this rank's algorithmic bytes
    # (16 B per state-update of its slab) over the step time.
    launches_per_step = launches / args.steps
    step_ms = ms / args.steps
    launch_bytes = 16.0 * 2 * n / world
    achieved = launch_bytes / (step_ms * 1e-3) / 1e9
    traffic = None
    kernel = heat_kernel_name(args.mode, args.grid)
    tp = os.path.join(ROOT, "profiles", "heat_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f).get(args.mode)
        if tj and tj.get("kernel") == kernel:
            traffic = tj["dram_bytes_per_update"] * 2 * n / world
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"CTMM heat3d grid={args.grid} (n={n}), embedding 2n, "
                               f"h={args.h}" + (f", z-slab sharded, {HALO_DESC[args.halo]}" if world > 1 else ""),
                   "mode": args.mode, "grid": args.grid, "n": n, "state_bytes": 32 * n,
                   "l2": "inputs (65.5 GB) far larger than the 126 MB L2; no flush needed",
                   "parallelism": f"zslab{world}"},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic, "peak_source": how,
                     "kernel": kernel, "algorithmic_bytes_per_launch": launch_bytes,
                     "avg_launch_ms": step_ms / max(1.0, launches_per_step) if world == 1 else None,
                     "per": "launch" if world == 1 else "step (per rank)",
                     "launches_per_step": launches_per_step},
        "finite": check["finite_ordered_bounded"],
        "check": check,
    }
    if args.mode == "fast" and not args.no_exact:
        # the bit-exact arithmetic mode on the same workload (reported beside the headline)
        import copy

        a2 = copy.copy(args)
        a2.mode = "exact"
        ms_e, _, clk_e, chk_e, _ = heat_device_bench(a2, world, rank, local, torch, pk, dist)
        line["exact_mode"] = {"value": updates / (ms_e * 1e-3), "ms_per_step": ms_e / args.steps,
                              "roofline_frac": (launch_bytes / (ms_e / args.steps * 1e-3) / 1e9) / hbm,
                              "clocks": clk_e, "check": chk_e}
    if not args.no_e2e and world == 1:
        e2e, ok2 = heat_e2e(args, pk, torch, world)
        line["e2e"] = e2e
        line["finite"] = line["finite"] and ok2
    elif not args.no_e2e:
        e2e = heat_e2e_sharded(args, pk, torch, dist, world, rank, local)
        if rank == 0:
            line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args)
    if rank == 0 and world == 1 and not args.no_secondary:
        line["secondary"] = secondary(args, pk, torch)
    if not args.no_secondary:  # configs 4 and 2 at N GPUs (the N = 1 values are their baselines)
        c4n = sharded_chain_bench(args, world, rank, local, torch, pk, dist)
        c2n = sharded_mc_bench(args, world, rank, local, torch, pk, dist)
        if rank == 0:
            line.setdefault("secondary", {})["C4_chain_sharded_nGPU"] = c4n
            line["secondary"]["C2_mc_sharded_nGPU"] = c2n
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------- reference arm

def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O

    import paper_2001_10635_b200 as pk

    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libivreach_ref.so not built"}))
        return
    g, per = args.cpu_grid, args.ref_steps_per_call
    model = pk.make_heat3d(g)
    n = g ** 3
    lo, hi = np.full(n, 0.9), np.full(n, 1.1)
    threads = O.ref_max_threads()
    rates, secs = [], 0.0
    for i in range(args.warmup + args.steps):
        r = O.ref_reach(O.METHOD_MM, model, lo, hi, None, None, 0.0, per * args.h, args.h, 0,
                        workers=threads, keep=False)
        if i >= args.warmup:
            secs += r.report["integration_s"]
            rates.append(2.0 * n * per / r.report["integration_s"])
    value = 2.0 * n * per * args.steps / secs
    sample = (f"ivreach::mixed_monotonicity heat3d grid={g} (n={n}), {per} RK4 steps per call, "
              f"h={args.h}; rate = 2n*steps/integration_s (the C5 grid=1600 needs 459 GB on CPU)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"CTMM heat3d (bounded sample grid={g} of the grid={GRID} workload)",
                       "parallelism": f"openmp{threads}"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": sample, **host_cpu()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def relaunch_under_torchrun(n):
    """`python bench.py --gpus N` without torchrun: re-exec as N ranks (one
    process per GPU, NCCL), the way the driver launches N > 1."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
           *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="fast", choices=["fast", "exact"])
    ap.add_argument("--grid", type=int, default=GRID)
    ap.add_argument("--h", type=float, default=H)
    ap.add_argument("--cpu-grid", type=int, default=300)
    ap.add_argument("--cpu-grid-max", type=int, default=800)
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--ref-steps-per-call", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-exact", action="store_true")
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process group backend for N > 1 (gloo: testing only, halos staged through the host)")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank on cuda:0 (tests the N > 1 code path on one GPU; with --backend gloo)")
    ap.add_argument("--chain-n", type=int, default=10 ** 7)
    ap.add_argument("--halo", default="peer", choices=["peer", "nccl"],
                    help="N > 1 heat halo transport: peer stores fused into the boundary launches "
                         "(CUDA IPC) or NCCL send/recv")
    ap.add_argument("--launcher-check", action="store_true",
                    help="print each rank's (rank, world) and exit: tests the --gpus relaunch without GPUs")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:
        relaunch_under_torchrun(args.gpus)
    if world and world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.launcher_check:
        w, r, lr = dist_env()
        print(json.dumps({"launcher_check": True, "rank": r, "local_rank": lr, "world": w,
                          "n_gpus": args.gpus}), flush=True)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
