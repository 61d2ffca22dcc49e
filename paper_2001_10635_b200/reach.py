"""Reference-facing API: the reachability entry points of
/root/reference/proj/include/ivreach/reach.hpp and the value types of
interval.hpp / system_model.hpp, executed by libpirk_b200.so on a B200.

Names, argument meaning and error behaviour follow the reference:
``std::invalid_argument`` -> ``ValueError``; ``std::runtime_error``
(IntegrationError, order violation, negative radius) -> ``RuntimeError``
with the reference's message text; ``std::bad_alloc`` -> ``MemoryError``.
A model the device library does not implement raises ``NotImplementedError``
(there is no CPU fallback).  ``workers`` keeps its reference meaning as a
parallelism request and must be >= 1; a single call runs on one GPU.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .models import SystemModel

# ------------------------------------------------------------- value types


class IntervalVector:
    """interval.hpp:13-28; validation of interval.cpp:10-23."""

    __slots__ = ("_lo", "_hi")

    def __init__(self, lower, upper, *, validate: bool = True):
        lo = np.ascontiguousarray(np.asarray(lower, dtype=np.float64).reshape(-1))
        hi = np.ascontiguousarray(np.asarray(upper, dtype=np.float64).reshape(-1))
        if validate:
            if lo.size != hi.size:
                raise ValueError(f"interval: lower has {lo.size} components, upper has {hi.size}")
            if lo.size == 0:
                raise ValueError("interval: dimension must be at least 1")
            fin = np.isfinite(lo) & np.isfinite(hi)
            if not fin.all():
                i = int(np.argmin(fin))
                raise ValueError(f"interval: non-finite bound at component {i}")
            bad = lo > hi
            if bad.any():
                raise ValueError(f"interval: lower > upper at component {int(np.argmax(bad))}")
        self._lo = lo
        self._hi = hi

    def dim(self) -> int:
        return int(self._lo.size)

    @property
    def lower(self) -> np.ndarray:
        return self._lo

    @property
    def upper(self) -> np.ndarray:
        return self._hi

    def __eq__(self, other) -> bool:
        return (isinstance(other, IntervalVector) and np.array_equal(self._lo, other._lo)
                and np.array_equal(self._hi, other._hi))

    def __repr__(self) -> str:
        return f"IntervalVector(dim={self.dim()})"


def center(box: IntervalVector) -> np.ndarray:
    return 0.5 * (box.upper + box.lower)  # interval.cpp:25-30


def half_width(box: IntervalVector) -> np.ndarray:
    return 0.5 * (box.upper - box.lower)  # interval.cpp:32-37


def from_center_radius(c, r) -> IntervalVector:
    """interval.cpp:39-53."""
    c = np.asarray(c, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    if c.size != r.size:
        raise ValueError(f"from_center_radius: center dim {c.size} != radius dim {r.size}")
    neg = r < 0.0
    if neg.any():
        raise ValueError(f"from_center_radius: negative radius at component {int(np.argmax(neg))}")
    return IntervalVector(c - r, c + r)


def contains(box: IntervalVector, x) -> bool:
    """interval.cpp:55-62."""
    x = np.asarray(x, dtype=np.float64)
    if x.size != box.dim():
        raise ValueError(f"contains: point dim {x.size} != box dim {box.dim()}")
    return bool(np.all((x >= box.lower) & (x <= box.upper)))


def subset_of(a: IntervalVector, b: IntervalVector) -> bool:
    """interval.cpp:81-88."""
    if a.dim() != b.dim():
        raise ValueError(f"subset_of: dim {a.dim()} != dim {b.dim()}")
    return bool(np.all((a.lower >= b.lower) & (a.upper <= b.upper)))


@dataclass
class ReachProblem:
    """system_model.hpp:47-55."""

    model: SystemModel
    initial: IntervalVector
    inputs: Optional[IntervalVector] = None
    t0: float = 0.0
    t1: float = 0.0
    h: float = 0.0
    tube_stride: int = 0


@dataclass
class MonteCarloSpec:
    """reach.hpp:55-60."""

    epsilon: float = 0.05
    delta: float = 0.01
    seed: int = 1
    samples_override: int = 0


@dataclass
class PhaseTimes:
    setup_s: float = 0.0
    integration_s: float = 0.0
    reduction_s: float = 0.0


@dataclass
class RunReport:
    """reach.hpp:19-30 (+ device accounting)."""

    method: str = ""
    n: int = 0
    m: int = 0
    workers: int = 1
    steps: int = 0
    peak_state_bytes: int = 0
    phases: PhaseTimes = field(default_factory=PhaseTimes)
    device_state_bytes: int = 0
    exact: bool = True
    kernel_launches: int = 0


@dataclass
class TubeEntry:
    t: float
    box: IntervalVector


@dataclass
class ReachTube:
    method: str
    entries: List[TubeEntry]
    report: RunReport

    def times(self) -> np.ndarray:
        return np.array([e.t for e in self.entries])


@dataclass
class StepPlan:
    full_steps: int
    has_remainder: bool

    def total(self) -> int:
        return self.full_steps + (1 if self.has_remainder else 0)


def validate(problem: ReachProblem) -> None:
    """system_model.cpp:10-32."""
    m = problem.model
    if m.dim == 0:
        raise ValueError("problem: model has no dynamics")
    if problem.initial.dim() != m.dim:
        raise ValueError(f"problem: initial box dim {problem.initial.dim()} does not match "
                         f"model dim {m.dim}")
    if m.input_dim == 0:
        if problem.inputs is not None:
            raise ValueError("problem: model has no inputs but an input box was given")
    else:
        if problem.inputs is None:
            raise ValueError(f"problem: model has {m.input_dim} inputs but no input box was given")
        if problem.inputs.dim() != m.input_dim:
            raise ValueError(f"problem: input box dim {problem.inputs.dim()} does not match "
                             f"model input dim {m.input_dim}")
    if not (problem.t0 < problem.t1):
        raise ValueError("problem: t0 must be earlier than t1")
    if not (problem.h > 0.0):
        raise ValueError("problem: step size h must be positive")


# ------------------------------------------------------------------ context

_EXC = {
    _lib.EINVAL: ValueError,
    _lib.EINTEGRATION: RuntimeError,
    _lib.EORDER: RuntimeError,
    _lib.ENEGRADIUS: RuntimeError,
    _lib.ENOMEM: MemoryError,
    _lib.ECUDA: RuntimeError,
    _lib.EUNSUPPORTED: NotImplementedError,
}


class Context:
    """A pirk_ctx: one arithmetic mode and one or more shard lanes (device +
    streams).  ``Context(0)`` is one lane on cuda:0; ``Context(devices=[0, 1,
    2, 3])`` shards chain / heat3d runs across four lanes (z-slabs / index
    ranges with NVLink halo copies) and Monte Carlo runs across their sample
    ranges -- bit-identical to one lane.  Device ids may repeat (lanes then
    share a GPU).  Calls on one context serialise on its mutex."""

    def __init__(self, device: int = 0, mode: str = "exact", devices=None):
        L = _lib.lib()
        h = C.c_void_p()
        devs = [int(device)] if devices is None else [int(d) for d in devices]
        arr = (C.c_int * len(devs))(*devs)
        st = L.pirk_create_multi(len(devs), arr, C.byref(h))
        if st != _lib.OK:
            raise RuntimeError(f"pirk_create(devices={devs}) failed with status {st} "
                               "(no CUDA device?)")
        self._h = h
        self.device = devs[0]
        self.devices = devs
        self._own_stream = L.pirk_get_stream(h)
        self.set_mode(mode)

    @property
    def lanes(self) -> int:
        return int(_lib.lib().pirk_lane_count(self._h))

    def set_record_callback(self, fn) -> None:
        """Stream recorded slots: ``fn(slot, step, t, lower, upper)`` (numpy
        views valid during the call; copy to keep) once per slot, in order,
        while the device integrates towards the next slot (pirk_c.h
        pirk_set_record_callback; the StepObserver of rk4.hpp:63-64).  None
        disables it.  With a callback the tube arrays may be skipped
        (``out=(None, None)`` is not needed: pass ``keep_tube=False``)."""
        if fn is None:
            self._record = None
            self.check(_lib.lib().pirk_set_record_callback(self._h, None, None))
            return

        def tramp(user, slot, step, t, lo, hi, n):
            lo_a = np.ctypeslib.as_array(lo, shape=(n,))
            hi_a = np.ctypeslib.as_array(hi, shape=(n,))
            fn(int(slot), int(step), float(t), lo_a, hi_a)

        self._record = _lib.RECORD_FN(tramp)  # keep the trampoline alive
        self.check(_lib.lib().pirk_set_record_callback(self._h, C.cast(self._record, C.c_void_p), None))

    def release_cache(self) -> None:
        """Free the state buffers kept for the next run of the same size."""
        self.check(_lib.lib().pirk_release_cache(self._h))

    @property
    def handle(self):
        return self._h

    def set_mode(self, mode: str) -> None:
        code = {"exact": _lib.MODE_EXACT, "fast": _lib.MODE_FAST}[mode]
        self.check(_lib.lib().pirk_set_mode(self._h, code))
        self.mode = mode

    def set_stream(self, stream_ptr: Optional[int]) -> None:
        """Launch on cudaStream_t ``stream_ptr`` (0 = the CUDA default stream);
        None restores the context's own stream."""
        if stream_ptr is None:
            stream_ptr = self._own_stream
        self.check(_lib.lib().pirk_set_stream(self._h, C.c_void_p(stream_ptr)))

    def launch_count(self) -> int:
        return int(_lib.lib().pirk_launch_count(self._h))

    def last_error(self) -> str:
        return _lib.lib().pirk_last_error(self._h).decode()

    def check(self, status: int) -> None:
        if status != _lib.OK:
            raise _EXC.get(status, RuntimeError)(self.last_error() or f"pirk status {status}")

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.lib().pirk_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_ctx_lock = threading.Lock()
_contexts: dict = {}
_default_mode = "exact"


def set_default_mode(mode: str) -> None:
    """'exact' (bit-identical to the reference) or 'fast' (FMA, <= 1e-12 rel.)."""
    global _default_mode
    if mode not in ("exact", "fast"):
        raise ValueError(f"unknown mode {mode!r}")
    _default_mode = mode


def get_context(device: int = 0) -> Context:
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = Context(device)
            _contexts[device] = ctx
    if ctx.mode != _default_mode:
        ctx.set_mode(_default_mode)
    return ctx


def lanes_for_workers(workers: int):
    """The reference's `workers` (reach.hpp:48,53,70) -> shard lanes: `workers`
    lanes spread round-robin over the visible GPUs (workers == device count
    puts one shard on each GPU)."""
    count = int(_lib.lib().pirk_device_count())
    if count == 0:
        raise RuntimeError("no CUDA device: the PIRK device library has no CPU fallback")
    return [r % count for r in range(int(workers))]


def get_worker_context(workers: int) -> Context:
    """Process-wide context for `workers` lanes (workers == 1: get_context())."""
    if workers <= 1:
        return get_context()
    with _ctx_lock:
        key = ("workers", int(workers))
        ctx = _contexts.get(key)
        if ctx is None:
            ctx = Context(devices=lanes_for_workers(workers))
            _contexts[key] = ctx
    if ctx.mode != _default_mode:
        ctx.set_mode(_default_mode)
    return ctx


# -------------------------------------------------------------- conversion

def model_struct(model: SystemModel) -> _lib.PirkModel:
    m = _lib.PirkModel()
    m.kind = int(model.kind)
    m.decomp = int(model.decomp)
    m.dim = int(model.dim)
    m.input_dim = int(model.input_dim)
    m.grid = int(model.grid)
    for i, v in enumerate(model.params):
        m.params[i] = float(v)
    if model.program is not None:
        m.program = model.program.handle
    return m


class _Marshalled:
    """Keeps the numpy buffers alive while the C structs point at them."""

    def __init__(self, problem: ReachProblem):
        self.lo = problem.initial.lower
        self.hi = problem.initial.upper
        self.plo = problem.inputs.lower if problem.inputs is not None else None
        self.phi = problem.inputs.upper if problem.inputs is not None else None
        p = _lib.PirkProblem()
        p.init_lower = _lib.dptr(self.lo)
        p.init_upper = _lib.dptr(self.hi)
        p.input_lower = _lib.dptr(self.plo)
        p.input_upper = _lib.dptr(self.phi)
        p.t0 = float(problem.t0)
        p.t1 = float(problem.t1)
        p.h = float(problem.h)
        p.tube_stride = int(problem.tube_stride)
        self.problem = p
        self.model = model_struct(problem.model)


def plan_steps(t0: float, t1: float, h: float) -> StepPlan:
    """rk4.cpp:8-17 (host arithmetic identical to the reference)."""
    full = C.c_uint64()
    rem = C.c_int32()
    st = _lib.lib().pirk_plan_steps(t0, t1, h, C.byref(full), C.byref(rem))
    if st != _lib.OK:
        if not (h > 0.0):
            raise ValueError("integrate: step size h must be positive")
        raise ValueError("integrate: t0 must be earlier than t1")
    return StepPlan(int(full.value), bool(rem.value))


def record_schedule(t0: float, t1: float, h: float, stride: int):
    """reach.cpp:28-39 -> (steps, times)."""
    L = _lib.lib()
    n = int(L.pirk_record_schedule(t0, t1, h, stride, None, None))
    steps = np.zeros(n, dtype=np.uint64)
    times = np.zeros(n)
    L.pirk_record_schedule(t0, t1, h, stride, steps.ctypes.data_as(C.POINTER(C.c_uint64)),
                           _lib.dptr(times))
    return steps, times


def sample_count(n: int, epsilon: float, delta: float) -> int:
    """reach.cpp:55-63."""
    if n == 0:
        raise ValueError("sample_count: n must be positive")
    if not (0.0 < epsilon < 1.0):
        raise ValueError("sample_count: epsilon must be in (0, 1)")
    if not (0.0 < delta < 1.0):
        raise ValueError("sample_count: delta must be in (0, 1)")
    out = C.c_uint64()
    _lib.lib().pirk_sample_count(n, epsilon, delta, C.byref(out))
    return int(out.value)


def _report(method: str, r: _lib.PirkReport, workers: int) -> RunReport:
    return RunReport(method=method, n=int(r.n), m=int(r.m), workers=workers, steps=int(r.steps),
                     peak_state_bytes=int(r.peak_state_bytes),
                     phases=PhaseTimes(r.setup_s, r.integration_s, r.reduction_s),
                     device_state_bytes=int(r.device_state_bytes), exact=bool(r.exact),
                     kernel_launches=int(r.kernel_launches))


def _alloc_tube(n: int, slots: int, out):
    if out is not None:
        lower, upper = out
        assert lower.dtype == np.float64 and upper.dtype == np.float64
        assert lower.size >= slots * n and upper.size >= slots * n
        return lower.reshape(-1)[: slots * n].reshape(slots, n), \
            upper.reshape(-1)[: slots * n].reshape(slots, n)
    return np.empty((slots, n)), np.empty((slots, n))


def _run_tube(fn_name: str, method: str, problem: ReachProblem, workers: int, ctx: Optional[Context],
              out, extra=()):
    validate(problem)
    if workers < 1:
        raise ValueError(f"{method.replace('-', '_')}: workers must be >= 1")
    ctx = ctx or get_worker_context(workers)
    mar = _Marshalled(problem)
    n = problem.model.dim
    _, times = record_schedule(problem.t0, problem.t1, problem.h, problem.tube_stride)
    slots = len(times)
    lower, upper = _alloc_tube(n, slots, out)
    tt = np.zeros(slots)
    tube = _lib.PirkTube()
    tube.times = _lib.dptr(tt)
    tube.lower = _lib.dptr(lower)
    tube.upper = _lib.dptr(upper)
    tube.max_slots = slots
    rep = _lib.PirkReport()
    fn = getattr(_lib.lib(), fn_name)
    ctx.check(fn(ctx.handle, C.byref(mar.model), C.byref(mar.problem), *extra, C.byref(tube),
                 C.byref(rep)))
    S = int(tube.n_slots)
    entries = [TubeEntry(float(tt[s]), IntervalVector(lower[s], upper[s], validate=False))
               for s in range(S)]
    return ReachTube(method, entries, _report(method, rep, workers))


# ------------------------------------------------------------ entry points

def growth_bound(problem: ReachProblem, workers: int = 1, *, ctx: Optional[Context] = None,
                 out=None) -> ReachTube:
    """reach.hpp:43-48 / reach.cpp:65-137."""
    if not problem.model.has_growth():
        validate(problem)
        raise ValueError("growth_bound: model has no deviation dynamics")
    return _run_tube("pirk_growth_bound", "growth-bound", problem, workers, ctx, out)


def mixed_monotonicity(problem: ReachProblem, workers: int = 1, *, ctx: Optional[Context] = None,
                       out=None) -> ReachTube:
    """reach.hpp:50-53 / reach.cpp:139-196."""
    if not problem.model.has_decomposition():
        validate(problem)
        raise ValueError("mixed_monotonicity: model has no decomposition function")
    return _run_tube("pirk_mixed_monotonicity", "mixed-monotonicity", problem, workers, ctx, out)


def monte_carlo(problem: ReachProblem, spec: MonteCarloSpec = MonteCarloSpec(), workers: int = 1,
                *, ctx: Optional[Context] = None, out=None) -> ReachTube:
    """reach.hpp:62-71 / reach.cpp:246-323."""
    if spec.samples_override == 0:
        sample_count(problem.model.dim, spec.epsilon, spec.delta)  # validates eps/delta
    s = _lib.PirkMcSpec(float(spec.epsilon), float(spec.delta), int(spec.seed),
                        int(spec.samples_override))
    tube = _run_tube("pirk_monte_carlo", "monte-carlo", problem, workers, ctx, out,
                     extra=(C.byref(s),))
    return tube


def monte_carlo_range(problem: ReachProblem, seed: int, s_begin: int, s_end: int,
                      lower: np.ndarray, upper: np.ndarray, *, ctx: Optional[Context] = None):
    """Fold samples [s_begin, s_end) into (lower, upper) (slots x n, caller
    initialised to +inf / -inf): one rank's share of a sample-sharded run."""
    validate(problem)
    ctx = ctx or get_context()
    mar = _Marshalled(problem)
    _, times = record_schedule(problem.t0, problem.t1, problem.h, problem.tube_stride)
    tube = _lib.PirkTube()
    tt = np.zeros(len(times))
    tube.times = _lib.dptr(tt)
    tube.lower = _lib.dptr(lower)
    tube.upper = _lib.dptr(upper)
    tube.max_slots = len(times)
    rep = _lib.PirkReport()
    ctx.check(_lib.lib().pirk_monte_carlo_range(ctx.handle, C.byref(mar.model),
                                                C.byref(mar.problem), int(seed), int(s_begin),
                                                int(s_end), C.byref(tube), C.byref(rep)))
    return tt


def coverage_estimate(problem: ReachProblem, spec: MonteCarloSpec, tube: ReachTube,
                      fresh_samples: int, seed: int, *, ctx: Optional[Context] = None) -> float:
    """reach.hpp:73-78 / reach.cpp:325-358."""
    validate(problem)
    if not tube.entries:
        raise ValueError("coverage_estimate: tube has no entries")
    if fresh_samples == 0:
        raise ValueError("coverage_estimate: fresh_samples must be positive")
    fin = tube.entries[-1].box
    if fin.dim() != problem.model.dim:
        raise ValueError("coverage_estimate: tube dimension mismatch")
    ctx = ctx or get_context()
    mar = _Marshalled(problem)
    frac = C.c_double()
    ctx.check(_lib.lib().pirk_coverage_estimate(ctx.handle, C.byref(mar.model),
                                                C.byref(mar.problem), _lib.dptr(fin.lower),
                                                _lib.dptr(fin.upper), int(fresh_samples),
                                                int(seed), C.byref(frac)))
    return float(frac.value)


def tube_to_csv(tube: ReachTube) -> str:
    """io.cpp:84-103 (``%.17g``)."""
    n = tube.entries[0].box.dim() if tube.entries else 0
    head = "t" + "".join(f",lower{i},upper{i}" for i in range(n))
    rows = [head]
    for e in tube.entries:
        parts = ["%.17g" % e.t]
        for lo, hi in zip(e.box.lower.tolist(), e.box.upper.tolist()):
            parts.append("%.17g" % lo)
            parts.append("%.17g" % hi)
        rows.append(",".join(parts))
    return "\n".join(rows) + "\n"


# ----------------------------------------------------------------- engine

class Engine:
    """Device-resident integrator (pirk_engine_*): the embedding (MM) or the
    growth-bound pair, advanced without host round trips.  Mirrors
    ivreach::Rk4Engine's reuse of state across steps (rk4.hpp:66-82)."""

    def __init__(self, problem: ReachProblem, method: str = "mixed-monotonicity",
                 ctx: Optional[Context] = None):
        validate(problem)
        self.ctx = ctx or get_context()
        self._mar = _Marshalled(problem)
        self.n = problem.model.dim
        code = {"mixed-monotonicity": _lib.METHOD_MM, "growth-bound": _lib.METHOD_GB}[method]
        h = C.c_void_p()
        self.ctx.check(_lib.lib().pirk_engine_create(self.ctx.handle, C.byref(self._mar.model),
                                                     code, C.byref(self._mar.problem),
                                                     C.byref(h)))
        self._h = h
        self.total_steps = plan_steps(problem.t0, problem.t1, problem.h).total()

    def advance(self, steps: int) -> None:
        self.ctx.check(_lib.lib().pirk_engine_advance(self._h, int(steps)))

    def status(self) -> int:
        done = C.c_uint64()
        self.ctx.check(_lib.lib().pirk_engine_status(self._h, C.byref(done)))
        return int(done.value)

    def read(self, lower: Optional[np.ndarray] = None, upper: Optional[np.ndarray] = None):
        lower = np.empty(self.n) if lower is None else lower
        upper = np.empty(self.n) if upper is None else upper
        self.ctx.check(_lib.lib().pirk_engine_read(self._h, _lib.dptr(lower), _lib.dptr(upper)))
        return lower, upper

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.lib().pirk_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def step_window(model: SystemModel, method: str, in0_ptr: int, in1_ptr: int, out0_ptr: int,
                out1_ptr: int, win_begin: int, win_len: int, out_begin: int, out_end: int,
                p0: Optional[Sequence[float]], p1: Optional[Sequence[float]], t: float, hk: float,
                step_index: int, fail_ptr: int = 0, *, ctx: Optional[Context] = None,
                mirror=None) -> None:
    """pirk_step_window on caller-owned device buffers (raw pointers).  With
    ``mirror=(lo0, lo1, lo_end, hi0, hi1, hi_begin)`` (pirk_step_window_mirror)
    output units u < lo_end are also stored to lo0/lo1 and units u >= hi_begin
    to hi0/hi1, indexed like out0/out1 (the neighbours' windows; a None
    pointer pair disables that side)."""
    ctx = ctx or get_context()
    m = model_struct(model)
    w = _lib.PirkWindow(in0_ptr, in1_ptr, out0_ptr, out1_ptr, win_begin, win_len, out_begin,
                        out_end)
    code = {"mixed-monotonicity": _lib.METHOD_MM, "growth-bound": _lib.METHOD_GB}[method]
    a0 = np.asarray(p0, dtype=np.float64) if p0 is not None else None
    a1 = np.asarray(p1, dtype=np.float64) if p1 is not None else None
    if mirror is None:
        ctx.check(_lib.lib().pirk_step_window(ctx.handle, C.byref(m), code, C.byref(w),
                                              _lib.dptr(a0), _lib.dptr(a1), float(t), float(hk),
                                              int(step_index), C.c_void_p(fail_ptr)))
    else:
        lo0, lo1, lo_end, hi0, hi1, hi_begin = mirror
        mr = _lib.PirkMirror(lo0, lo1, int(lo_end) if lo0 else 0, hi0, hi1, int(hi_begin) if hi0 else 0)
        ctx.check(_lib.lib().pirk_step_window_mirror(
            ctx.handle, C.byref(m), code, C.byref(w), C.byref(mr),
            _lib.dptr(a0), _lib.dptr(a1), float(t), float(hk), int(step_index), C.c_void_p(fail_ptr)))
