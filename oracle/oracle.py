"""ctypes access to the parity checkers -- TEST INFRASTRUCTURE ONLY.

Two CPU implementations of the reference hot path:

* ``restatement`` -- oracle/build/libpirk_oracle.so, the plain-C restatement
  (oracle/pirk_oracle.c, every function cites /root/reference/proj file:line);
* ``reference``   -- oracle/_ref/libivreach_ref.so, the unmodified reference
  sources (/root/reference/proj/src) compiled by oracle/Makefile behind
  oracle/ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  The product package
(paper_2001_10635_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "libpirk_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libivreach_ref.so")

METHOD_MM, METHOD_GB, METHOD_MC = 0, 1, 2


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class PoModel(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("decomp", C.c_int32),
        ("dim", C.c_uint64),
        ("input_dim", C.c_uint64),
        ("grid", C.c_uint64),
        ("params", C.c_double * 8),
    ]


def to_po(model) -> PoModel:
    """Accepts any object with kind/decomp/dim/input_dim/grid/params attributes
    (e.g. paper_2001_10635_b200.SystemModel)."""
    m = PoModel()
    m.kind = int(model.kind)
    m.decomp = int(model.decomp)
    m.dim = int(model.dim)
    m.input_dim = int(model.input_dim)
    m.grid = int(getattr(model, "grid", 0) or 0)
    for i, v in enumerate(model.params):
        m.params[i] = float(v)
    return m


_DP = C.POINTER(C.c_double)
_U64P = C.POINTER(C.c_uint64)


def _dp(a):
    if a is None:
        return None
    return a.ctypes.data_as(_DP)


def _arr(x, n=None):
    if x is None:
        return None
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if n is not None and a.size == 1 and n > 1:
        a = np.full(n, float(a.reshape(-1)[0]))
    return a


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            raise OSError(f"oracle not built: {ORACLE_SO} (run make -C oracle)")
        L = C.CDLL(ORACLE_SO)
        L.po_u01.restype = C.c_double
        L.po_u01.argtypes = [C.c_uint64] * 3
        L.po_mix64.restype = C.c_uint64
        L.po_mix64.argtypes = [C.c_uint64]
        L.po_plan_steps.argtypes = [C.c_double, C.c_double, C.c_double, _U64P, C.POINTER(C.c_int)]
        L.po_record_schedule.restype = C.c_uint64
        L.po_record_schedule.argtypes = [C.c_double, C.c_double, C.c_double, C.c_uint64, _U64P, _DP]
        L.po_sample_count.argtypes = [C.c_uint64, C.c_double, C.c_double, _U64P]
        for name in ("po_rhs", "po_growth"):
            f = getattr(L, name)
            f.restype = C.c_double
            f.argtypes = [C.POINTER(PoModel), C.c_uint64, C.c_double, _DP, _DP]
        L.po_decomp.restype = C.c_double
        L.po_decomp.argtypes = [C.POINTER(PoModel), C.c_uint64, C.c_double, _DP, _DP, _DP, _DP]
        L.po_growth_matrix.argtypes = [C.POINTER(PoModel), _DP]
        L.po_integrate.argtypes = [C.POINTER(PoModel), _DP, _DP, C.c_double, C.c_double,
                                   C.c_double, C.c_uint64, _DP, _DP, _U64P, _U64P, _DP]
        sig = [C.POINTER(PoModel), _DP, _DP, _DP, _DP, C.c_double, C.c_double, C.c_double,
               C.c_uint64, _DP, _DP, _DP, C.c_char_p, C.c_int]
        L.po_mixed_monotonicity.argtypes = sig
        L.po_growth_bound.argtypes = sig
        L.po_monte_carlo.argtypes = [C.POINTER(PoModel), _DP, _DP, _DP, _DP, C.c_double,
                                     C.c_double, C.c_double, C.c_uint64, C.c_uint64,
                                     C.c_uint64, C.c_uint64, _DP, _DP, _DP, C.c_char_p, C.c_int]
        L.po_coverage_estimate.argtypes = [C.POINTER(PoModel), _DP, _DP, _DP, _DP, C.c_double,
                                           C.c_double, C.c_double, _DP, _DP, C.c_uint64,
                                           C.c_uint64, _DP]
        L.po_step_window.argtypes = [C.POINTER(PoModel), C.c_int, _DP, _DP, _DP, _DP,
                                     C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _DP, _DP,
                                     C.c_double, C.c_double]
        _lib = L
    return _lib


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise OSError(f"reference oracle not built: {REF_SO} (run make -C oracle ref)")
        L = C.CDLL(REF_SO)
        L.ref_u01.restype = C.c_double
        L.ref_u01.argtypes = [C.c_uint64] * 3
        L.ref_max_threads.restype = C.c_int
        L.ref_sample_count.argtypes = [C.c_uint64, C.c_double, C.c_double, _U64P]
        L.ref_plan_steps.argtypes = [C.c_double, C.c_double, C.c_double, _U64P, C.POINTER(C.c_int)]
        L.ref_eval.argtypes = [C.POINTER(PoModel), C.c_int, C.c_double, _DP, _DP, _DP, _DP, _DP,
                               C.c_char_p, C.c_int]
        L.ref_integrate.argtypes = [C.POINTER(PoModel), _DP, _DP, C.c_double, C.c_double,
                                    C.c_double, C.c_uint64, _DP, _DP, C.c_uint64, _U64P,
                                    C.c_char_p, C.c_int]
        L.ref_reach.argtypes = [C.POINTER(PoModel), C.c_int, _DP, _DP, _DP, _DP, C.c_double,
                                C.c_double, C.c_double, C.c_uint64, C.c_int, C.c_uint64,
                                C.c_uint64, C.c_double, C.c_double, _DP, _DP, _DP, C.c_uint64,
                                _U64P, _U64P, _DP, _DP, C.c_char_p, C.c_int]
        L.ref_coverage.argtypes = [C.POINTER(PoModel), _DP, _DP, _DP, _DP, C.c_double,
                                   C.c_double, C.c_double, _DP, _DP, C.c_uint64, C.c_uint64,
                                   _DP, C.c_char_p, C.c_int]
        _ref = L
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_SO)


# ----------------------------------------------------------------- helpers

def u01(seed, stream, index):
    return lib().po_u01(seed, stream, index)


def _mix64(z):
    """rng.hpp:11-16 on uint64 arrays (wrapping arithmetic)."""
    z = z + np.uint64(0x9e3779b97f4a7c15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xbf58476d1ce4e5b9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94d049bb133111eb)
    return z ^ (z >> np.uint64(31))


def u01_vec(seed, stream, index):
    """rng.hpp:19-23 u01(seed, stream, index) vectorised over `index` (for
    inputs of 1e7 components, where the per-call ctypes path is too slow)."""
    with np.errstate(over="ignore"):
        idx = np.asarray(index, dtype=np.uint64)
        a = _mix64(np.uint64(seed)) ^ (np.uint64(stream) * np.uint64(0xd1342543de82ef95))
        z = _mix64(_mix64(a) ^ (idx * np.uint64(0xaf251af3b0f025b5)))
        return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def plan_steps(t0, t1, h):
    full = C.c_uint64()
    rem = C.c_int()
    rc = lib().po_plan_steps(t0, t1, h, C.byref(full), C.byref(rem))
    if rc:
        raise OracleError(rc, "plan_steps: invalid arguments")
    return int(full.value), bool(rem.value)


def record_schedule(t0, t1, h, stride):
    n = lib().po_record_schedule(t0, t1, h, stride, None, None)
    steps = np.zeros(n, dtype=np.uint64)
    times = np.zeros(n)
    lib().po_record_schedule(t0, t1, h, stride, steps.ctypes.data_as(_U64P), _dp(times))
    return steps, times


def sample_count(n, eps, delta):
    out = C.c_uint64()
    rc = lib().po_sample_count(n, eps, delta, C.byref(out))
    if rc:
        raise OracleError(rc, "sample_count: invalid arguments")
    return int(out.value)


def eval_field(model, which, x, p=None, xh=None, ph=None, t=0.0):
    """which: 'rhs' | 'growth' | 'decomp'. Returns the full vector."""
    m = to_po(model)
    n = int(model.dim)
    x = _arr(x)
    p = _arr(p if p is not None else np.zeros(max(1, int(model.input_dim))))
    out = np.empty(n)
    L = lib()
    for i in range(n):
        if which == "rhs":
            out[i] = L.po_rhs(C.byref(m), i, t, _dp(x), _dp(p))
        elif which == "growth":
            out[i] = L.po_growth(C.byref(m), i, t, _dp(x), _dp(p))
        else:
            xh_ = _arr(xh)
            ph_ = _arr(ph if ph is not None else p)
            out[i] = L.po_decomp(C.byref(m), i, t, _dp(x), _dp(p), _dp(xh_), _dp(ph_))
    return out


def growth_matrix(model):
    n = int(model.dim)
    Cm = np.zeros(n * n)
    m = to_po(model)
    if not lib().po_growth_matrix(C.byref(m), _dp(Cm)):
        return None
    return Cm.reshape(n, n)


@dataclass
class OracleTube:
    times: np.ndarray
    lower: np.ndarray  # slots x n
    upper: np.ndarray


def _inputs(model, plo, phi):
    ni = int(model.input_dim)
    if ni == 0:
        return None, None
    return _arr(plo, ni), _arr(phi, ni)


def integrate(model, x0, p, t0, t1, h, stride=0):
    m = to_po(model)
    n = int(model.dim)
    _, times = record_schedule(t0, t1, h, stride)
    states = np.zeros((len(times), n))
    es, ec, et = C.c_uint64(), C.c_uint64(), C.c_double()
    p = _arr(p if p is not None else [0.0])
    rc = lib().po_integrate(C.byref(m), _dp(_arr(x0, n)), _dp(p), t0, t1, h, stride,
                            _dp(times), _dp(states), C.byref(es), C.byref(ec), C.byref(et))
    if rc:
        raise OracleError(rc, f"integration produced a non-finite value at step {es.value}, "
                              f"component {ec.value}, t = {et.value:f}")
    return times, states


def _method(fn, model, lo, hi, plo, phi, t0, t1, h, stride):
    n = int(model.dim)
    m = to_po(model)
    lo, hi = _arr(lo, n), _arr(hi, n)
    plo, phi = _inputs(model, plo, phi)
    _, times = record_schedule(t0, t1, h, stride)
    S = len(times)
    out_lo = np.zeros((S, n))
    out_hi = np.zeros((S, n))
    tt = np.zeros(S)
    err = C.create_string_buffer(512)
    rc = fn(C.byref(m), _dp(lo), _dp(hi), _dp(plo), _dp(phi), t0, t1, h, stride, _dp(tt),
            _dp(out_lo), _dp(out_hi), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return OracleTube(tt, out_lo, out_hi)


def mixed_monotonicity(model, lo, hi, plo, phi, t0, t1, h, stride=0):
    return _method(lib().po_mixed_monotonicity, model, lo, hi, plo, phi, t0, t1, h, stride)


def growth_bound(model, lo, hi, plo, phi, t0, t1, h, stride=0):
    return _method(lib().po_growth_bound, model, lo, hi, plo, phi, t0, t1, h, stride)


def monte_carlo(model, lo, hi, plo, phi, t0, t1, h, stride, seed, samples, s_begin=0,
                s_end=None):
    n = int(model.dim)
    m = to_po(model)
    lo, hi = _arr(lo, n), _arr(hi, n)
    plo, phi = _inputs(model, plo, phi)
    _, times = record_schedule(t0, t1, h, stride)
    S = len(times)
    out_lo = np.full((S, n), np.inf)
    out_hi = np.full((S, n), -np.inf)
    tt = np.zeros(S)
    err = C.create_string_buffer(512)
    s_end = samples if s_end is None else s_end
    rc = lib().po_monte_carlo(C.byref(m), _dp(lo), _dp(hi), _dp(plo), _dp(phi), t0, t1, h,
                              stride, seed, s_begin, s_end, _dp(tt), _dp(out_lo),
                              _dp(out_hi), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return OracleTube(tt, out_lo, out_hi)


def coverage_estimate(model, lo, hi, plo, phi, t0, t1, h, box_lo, box_hi, fresh, seed):
    n = int(model.dim)
    m = to_po(model)
    plo, phi = _inputs(model, plo, phi)
    frac = C.c_double()
    rc = lib().po_coverage_estimate(C.byref(m), _dp(_arr(lo, n)), _dp(_arr(hi, n)), _dp(plo),
                                    _dp(phi), t0, t1, h, _dp(_arr(box_lo, n)),
                                    _dp(_arr(box_hi, n)), fresh, seed, C.byref(frac))
    if rc:
        raise OracleError(rc, "coverage_estimate failed")
    return frac.value


def step_window(model, method, in0, in1, win_begin, win_len, out_begin, out_end, p0, p1, t,
                hk):
    """One windowed RK4 step (see pirk_oracle.h po_step_window)."""
    m = to_po(model)
    unit = int(model.grid) ** 2 if int(model.kind) == 4 else 1
    cnt = (out_end - out_begin) * unit
    o0 = np.empty(cnt)
    o1 = np.empty(cnt)
    p0 = _arr(p0) if p0 is not None else None
    p1 = _arr(p1) if p1 is not None else None
    rc = lib().po_step_window(C.byref(m), method, _dp(_arr(in0)), _dp(_arr(in1)), _dp(o0),
                              _dp(o1), win_begin, win_len, out_begin, out_end, _dp(p0),
                              _dp(p1), t, hk)
    if rc:
        raise OracleError(rc, "step_window: bad window")
    return o0, o1


# --------------------------------------------------- the reference itself

@dataclass
class RefResult:
    times: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    report: dict
    wall_s: float


def ref_reach(method, model, lo, hi, plo, phi, t0, t1, h, stride=0, workers=1, samples=0,
              seed=1, eps=0.05, delta=0.01, keep=True):
    """Run the reference's own mixed_monotonicity / growth_bound / monte_carlo."""
    n = int(model.dim)
    m = to_po(model)
    lo, hi = _arr(lo, n), _arr(hi, n)
    plo, phi = _inputs(model, plo, phi)
    _, times = record_schedule(t0, t1, h, stride)
    S = len(times)
    out_lo = np.zeros((S, n)) if keep else None
    out_hi = np.zeros((S, n)) if keep else None
    tt = np.zeros(S)
    ns = C.c_uint64()
    rep = np.zeros(4, dtype=np.uint64)
    ph = np.zeros(3)
    wall = C.c_double()
    err = C.create_string_buffer(1024)
    rc = ref_lib().ref_reach(C.byref(m), method, _dp(lo), _dp(hi), _dp(plo), _dp(phi), t0, t1,
                             h, stride, workers, samples, seed, eps, delta, _dp(tt),
                             _dp(out_lo), _dp(out_hi), S, C.byref(ns),
                             rep.ctypes.data_as(_U64P), _dp(ph), C.byref(wall), err, 1024)
    if rc:
        raise OracleError(rc, err.value.decode())
    report = {"n": int(rep[0]), "m": int(rep[1]), "steps": int(rep[2]),
              "peak_state_bytes": int(rep[3]), "setup_s": ph[0], "integration_s": ph[1],
              "reduction_s": ph[2]}
    return RefResult(tt[: ns.value], out_lo, out_hi, report, wall.value)


def ref_eval(model, which, x, p=None, xh=None, ph=None, t=0.0):
    m = to_po(model)
    n = int(model.dim)
    w = {"rhs": 0, "growth": 1, "decomp": 2}[which]
    out = np.empty(n)
    err = C.create_string_buffer(512)
    x = _arr(x)
    p = _arr(p) if p is not None else None
    xh = _arr(xh) if xh is not None else None
    ph = _arr(ph) if ph is not None else None
    rc = ref_lib().ref_eval(C.byref(m), w, t, _dp(x), _dp(p), _dp(xh), _dp(ph), _dp(out), err,
                            512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return out


def ref_max_threads():
    return ref_lib().ref_max_threads()


# ------------------------------------------ uniform-box heat3d: the 1-D line

def heat_line_uniform(g, value, steps, h, alpha=1.0, exchange=1.0, t0=0.0):
    """heat3d (models.cpp:92-133) from a box that is uniform in every component,
    in exact reference arithmetic, for ANY grid -- including C5's g = 1600.

    Only the x = 0 face exchanges heat (Robin ghost, models.cpp:116-119); the
    y and z faces are insulated (:121-125).  A field that is constant over
    every (y, z) plane therefore stays so: each y/z stencil term is
    ``x[i -+ g] - self == 0.0`` exactly, and ``acc + 0.0 == acc`` (up to the
    sign of a zero, which == ignores).  Every component of the g^3 field
    equals the 1-D line computed here with the reference's expression order:
    acc = (x- term) + (x+ term), f = k*acc, and the RK4 update of rk4.cpp:38-68
    (u = x + h2*k, x + h6*(((k0 + 2k1) + 2k2) + k3)), with the step plan of
    rk4.cpp:8-17 / :99-100 for t1 = t0 + steps*h.  numpy's elementwise float64
    add/mul are single IEEE operations (no contraction), so the result is
    bit-exact.  Returns the line after `steps` steps (index = ix).
    """
    delta = 1.0 / float(g - 1)
    k = alpha / (delta * delta)
    robin = 2.0 * delta * exchange

    def f(x):
        acc = np.zeros_like(x)
        acc[1:] = acc[1:] + (x[:-1] - x[1:])
        acc[0] = acc[0] + ((x[1] - x[0]) - robin * x[0])
        acc[:-1] = acc[:-1] + (x[1:] - x[:-1])
        return k * acc

    x = np.full(g, float(value))
    plan = []
    t1 = t0 + steps * h
    span = t1 - t0
    full = int(np.floor(span / h + 1e-9))
    rem = span - float(full) * h
    total = full + (1 if rem > 1e-9 * h else 0)
    for kk in range(total):
        t = t0 + float(kk) * h
        plan.append((t1 - t) if kk + 1 == total else h)
    for hk in plan:
        h2 = 0.5 * hk
        h6 = hk / 6.0
        k0 = f(x)
        k1 = f(x + h2 * k0)
        k2 = f(x + h2 * k1)
        k3 = f(x + hk * k2)
        x = x + h6 * (((k0 + 2.0 * k1) + 2.0 * k2) + k3)
    return x
