"""Config-file front end routed to the GPU path.

Restates the reference's run-configuration layer so a ``.cfg`` file written
for ``ivreach run`` drives the device library unchanged:

* ``parse_config`` / ``parse_config_file``  config.cpp:95-270 (same keys, scalar
  broadcast of box entries, catalog defaults, the same invalid_argument
  messages with line numbers -> ValueError);
* ``serialize_config``                      config.cpp:272-291;
* the model catalog the parser resolves against  models.cpp:694-1000
  (``find_model``, ``resolve_params`` :1022-1032, parameter defaults, the
  methods each model supports, default problems);
* ``build_problem`` / ``run_config``        driver.cpp:43-72, dispatching to
  the device entry points and writing the tube and report files in the
  reference's formats (io.cpp, via driver.py).

``workers`` (0 = all) maps to shard lanes: 0 means one lane per visible GPU.
Catalog models without a device kernel (quadrotor-swarm, quadrotor-apf,
single-track -- out of scope) parse exactly as in the reference
but ``run_config`` rejects them.
"""
from __future__ import annotations

import math
import os
import re
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Tuple

from . import models as M
from .reach import IntervalVector, MonteCarloSpec, ReachProblem, validate

KGRAVITY = 9.81


@dataclass
class ParamSpec:
    name: str
    value: float


@dataclass
class CatalogEntry:
    """ModelCatalogEntry (models.hpp:110-121), the parts the front end uses."""

    name: str
    methods: List[str]
    params: List[ParamSpec]
    dims: Callable[[Dict[str, float]], Tuple[int, int]]  # (dim, input_dim)
    make: Optional[Callable[[Dict[str, float]], M.SystemModel]]  # None: no device kernel
    default_problem: Callable[[int, Dict[str, float]], tuple]  # (lo, hi, plo, phi, t1, h)


def _at(p: Dict[str, float], name: str) -> float:
    return p[name]


def _count_at(p: Dict[str, float], name: str) -> int:
    """models.cpp:677-684."""
    v = p[name]
    if v < 0 or v != math.floor(v):
        raise ValueError(f"parameter {name} must be a nonnegative integer, got {v:f}")
    return int(v)


_ALL3 = ["growth-bound", "mixed-monotonicity", "monte-carlo"]
_GB_MC = ["growth-bound", "monte-carlo"]


def _fill(n, lo, hi):
    return [lo] * n, [hi] * n


def _tile(k, lo, hi):
    return lo * k, hi * k


def _swarm_default(n, p):
    k = n // 12
    hover = p["mass"] * p["gravity"]
    lo, hi = _tile(k, [-0.1] * 6 + [-0.05] * 6, [0.1] * 6 + [0.05] * 6)
    plo, phi = _tile(k, [hover - 0.15, -0.01, -0.01, -0.01], [hover + 0.15, 0.01, 0.01, 0.01])
    return lo, hi, plo, phi, 1.0, 0.01


def _apf_default(n, p):
    k = n // 12
    hover = p["mass"] * p["gravity"]
    lo, hi = [], []
    for q in range(k):
        base = 2.0 * float(q)
        lo += [base - 0.1, -0.1, -0.1, -0.1, -0.1, -0.1] + [-0.05] * 6
        hi += [base + 0.1, 0.1, 0.1, 0.1, 0.1, 0.1] + [0.05] * 6
    plo, phi = _tile(k, [hover - 0.15, -0.01, -0.01, -0.01], [hover + 0.15, 0.01, 0.01, 0.01])
    return lo, hi, plo, phi, 1.0, 0.01


_QUAD = [("mass", 1.4), ("gravity", KGRAVITY), ("jx", 0.054), ("jy", 0.054), ("jz", 0.104)]

CATALOG_ENTRIES: List[CatalogEntry] = [
    CatalogEntry(
        "traffic", _ALL3,
        [ParamSpec(*t) for t in [("segments", 50), ("v", 0.5), ("w", 1.0 / 6.0), ("c", 40), ("xbar", 320),
                                 ("period", 30), ("beta", 0.75)]],
        lambda p: (_count_at(p, "segments"), 1),
        lambda p: M.make_traffic(_count_at(p, "segments"), p["v"], p["w"], p["c"], p["xbar"], p["period"],
                                 p["beta"]),
        lambda n, p: (*_fill(n, 10.0, 20.0), [4.0], [6.0], 30.0, 0.5)),
    CatalogEntry(
        "heat3d", _ALL3,
        [ParamSpec(*t) for t in [("grid", 8), ("alpha", 1.0), ("exchange", 1.0)]],
        lambda p: (_count_at(p, "grid") ** 3, 0),
        lambda p: M.make_heat3d(_count_at(p, "grid"), p["alpha"], p["exchange"]),
        lambda n, p: (*_fill(n, 0.9, 1.1), None, None, 0.05, 0.002)),
    CatalogEntry(
        "quadrotor-swarm", _GB_MC,
        [ParamSpec(*t) for t in [("quadrotors", 2), ("thrust_bound", 27.5)] + _QUAD],
        lambda p: (12 * _count_at(p, "quadrotors"), 4 * _count_at(p, "quadrotors")),
        None, _swarm_default),
    CatalogEntry(
        "quadrotor-apf", _GB_MC,
        [ParamSpec(*t) for t in [("quadrotors", 2), ("f_repel", 1.0), ("f_attract", 1.0),
                                 ("thrust_bound", 27.5)] + _QUAD],
        lambda p: (12 * _count_at(p, "quadrotors"), 4 * _count_at(p, "quadrotors")),
        None, _apf_default),
    CatalogEntry(
        "single-track", _GB_MC,
        [ParamSpec(*t) for t in [("lwb", 2.5789), ("mass", 1093.3), ("mu", 1.0489), ("lf", 1.156),
                                 ("lr", 1.422), ("hcg", 0.6137), ("iz", 1791.6), ("csf", 20.89),
                                 ("csr", 20.89), ("gravity", KGRAVITY), ("delta_min", -1.066),
                                 ("delta_max", 1.066), ("vdelta_min", -0.4), ("vdelta_max", 0.4),
                                 ("v_min", -13.6), ("v_max", 50.8), ("v_switch", 7.319), ("a_max", 11.5),
                                 ("op_v_lo", 5.0), ("op_x3", 0.2), ("op_x6", 1.0), ("op_x7", 0.3)]],
        lambda p: (7, 2), None,
        lambda n, p: ([-0.1, -0.1, 0.0, 14.9, -0.05, 0.0, 0.0], [0.1, 0.1, 0.0, 15.1, 0.05, 0.0, 0.0],
                      [0.0, 0.0], [0.0, 0.0], 1.0, 0.005)),
    CatalogEntry(
        "vdp", _GB_MC, [ParamSpec(*t) for t in [("mu", 1.0), ("op_x", 2.5), ("op_y", 3.0)]],
        lambda p: (2, 0), lambda p: M.make_vdp(p["mu"], p["op_x"], p["op_y"]),
        lambda n, p: ([1.25, 2.35], [1.55, 2.45], None, None, 1.0, 0.005)),
    CatalogEntry(
        "laub-loomis", _GB_MC, [], lambda p: (7, 0), lambda p: M.make_laub_loomis(),
        lambda n, p: ([c - 0.05 for c in (1.2, 1.05, 1.5, 2.4, 1.0, 0.1, 0.45)],
                      [c + 0.05 for c in (1.2, 1.05, 1.5, 2.4, 1.0, 0.1, 0.45)], None, None, 1.0, 0.005)),
    CatalogEntry(
        "arch-quadrotor", _GB_MC, [ParamSpec(*t) for t in _QUAD], lambda p: (12, 0),
        lambda p: M.make_arch_quadrotor(p["mass"], p["gravity"], p["jx"], p["jy"], p["jz"]),
        lambda n, p: ([-0.4] * 6 + [0.0] * 6, [0.4] * 6 + [0.0] * 6, None, None, 1.0, 0.01)),
    CatalogEntry(
        "zero", _ALL3, [ParamSpec("dim", 2)], lambda p: (_count_at(p, "dim"), 0),
        lambda p: M.make_zero(_count_at(p, "dim")),
        lambda n, p: (*_fill(n, 0.0, 1.0), None, None, 1.0, 0.1)),
    CatalogEntry(
        "scalar-decay", _ALL3, [], lambda p: (1, 1), lambda p: M.make_scalar_decay(),
        lambda n, p: ([0.9], [1.1], [0.0], [0.0], 1.0, 0.001)),
    CatalogEntry(
        "scalar-linear", _ALL3, [ParamSpec("a", 1.0)], lambda p: (1, 0),
        lambda p: M.make_scalar_linear(p["a"]),
        lambda n, p: ([1.0], [2.0], None, None, 1.0, 0.001)),
]


def find_model(name: str) -> Optional[CatalogEntry]:
    """models.cpp:1010-1020."""
    for e in CATALOG_ENTRIES:
        if e.name == name:
            return e
    return None


def resolve_params(entry: CatalogEntry, overrides: Dict[str, float]) -> Dict[str, float]:
    """models.cpp:1022-1032 (std::map: name order)."""
    out = {s.name: float(s.value) for s in entry.params}
    for name, value in overrides.items():
        if name not in out:
            raise ValueError(f"model {entry.name} has no parameter named {name}")
        out[name] = float(value)
    return dict(sorted(out.items()))


@dataclass
class RunConfig:
    """config.hpp:14-32."""

    model: str = ""
    params: Dict[str, float] = field(default_factory=dict)
    method: str = ""
    initial_lower: List[float] = field(default_factory=list)
    initial_upper: List[float] = field(default_factory=list)
    input_lower: List[float] = field(default_factory=list)
    input_upper: List[float] = field(default_factory=list)
    t0: float = 0.0
    t1: float = 0.0
    h: float = 0.0
    tube_stride: int = 0
    workers: int = 0
    epsilon: float = 0.05
    delta: float = 0.01
    seed: int = 1
    samples: int = 0
    output: str = "ivreach-out"
    format: str = "json"


_SCALAR_KEYS = ("model", "method", "initial.lower", "initial.upper", "input.lower", "input.upper", "t0",
                "t1", "h", "tube_stride", "workers", "epsilon", "delta", "seed", "samples", "output",
                "format")
_METHODS = ["growth-bound", "mixed-monotonicity", "monte-carlo"]
_FLOAT = re.compile(r"[+-]?((\d+\.?\d*|\.\d+)([eE][+-]?\d+)?|inf(inity)?|nan(\([0-9A-Za-z_]*\))?)", re.I)
_HEXF = re.compile(r"[+-]?0[xX]([0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)([pP][+-]?\d+)?")


def _fail(line: int, msg: str):
    raise ValueError(f"config line {line}: {msg}")


def _trim(s: str) -> str:
    return s.strip(" \t\n\r\f\v")


def _parse_double(value: str, key: str, line: int) -> float:
    """config.cpp:27-34: strtod over the whole trimmed value."""
    v = _trim(value)
    if _FLOAT.fullmatch(v):
        return float(v)
    if _HEXF.fullmatch(v):
        return float.fromhex(v)
    _fail(line, f"invalid number '{v}' for key '{key}'")


def _parse_uint(value: str, key: str, line: int) -> int:
    """config.cpp:36-45: strtoull, no sign."""
    v = _trim(value)
    if not v or v[0] == "-" or not re.fullmatch(r"\+?\d+", v):
        _fail(line, f"invalid nonnegative integer '{v}' for key '{key}'")
    return min(int(v), (1 << 64) - 1)


def _parse_vector(value: str, key: str, line: int) -> List[float]:
    """config.cpp:47-55 (std::getline on ',': a trailing empty item is dropped)."""
    items = value.split(",")
    if items and items[-1] == "":
        items = items[:-1]
    out = [_parse_double(it, key, line) for it in items]
    if not out:
        _fail(line, f"empty value for key '{key}'")
    return out


def _resolve_box_side(raw, key, want, model, what):
    """config.cpp:87-96."""
    v = _parse_vector(raw[0], key, raw[1])
    if len(v) == 1 and want > 1:
        return [v[0]] * want
    if len(v) != want:
        _fail(raw[1], f"{key} has {len(v)} entries but model '{model}' has {what} {want}")
    return v


def parse_config(text: str) -> RunConfig:
    """config.cpp:100-262."""
    kv: Dict[str, tuple] = {}
    param_kv: Dict[str, tuple] = {}
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()  # std::getline yields no final empty line after a trailing newline
    for lineno, full in enumerate(lines, start=1):
        body = _trim(full.split("#", 1)[0])
        if not body:
            continue
        if "=" not in body:
            _fail(lineno, "expected 'key = value'")
        key, value = body.split("=", 1)
        key, value = _trim(key), _trim(value)
        if not key:
            _fail(lineno, "expected 'key = value'")
        if key.startswith("param."):
            name = key[6:]
            if not name:
                _fail(lineno, "empty parameter name")
            param_kv[name] = (value, lineno)
            continue
        if key not in _SCALAR_KEYS:
            _fail(lineno, f"unknown key '{key}'")
        kv[key] = (value, lineno)

    cfg = RunConfig()
    if "model" not in kv:
        raise ValueError("config: missing required key 'model'")
    cfg.model = _trim(kv["model"][0])
    entry = find_model(cfg.model)
    if entry is None:
        _fail(kv["model"][1], f"unknown model '{cfg.model}'")
    overrides = {}
    for name in sorted(param_kv):
        value, line = param_kv[name]
        if name not in {s.name for s in entry.params}:
            _fail(line, f"model '{cfg.model}' has no parameter named '{name}'")
        overrides[name] = _parse_double(value, "param." + name, line)
    cfg.params = resolve_params(entry, overrides)
    try:
        dim, input_dim = entry.dims(cfg.params)
        if entry.make is not None:
            entry.make(cfg.params)  # the catalog constructor's validation
    except ValueError as e:
        raise ValueError("config: " + str(e)) from None

    if "method" in kv:
        cfg.method = _trim(kv["method"][0])
        if cfg.method not in _METHODS:
            _fail(kv["method"][1], f"unknown method '{cfg.method}' (expected {', '.join(_METHODS)})")
        if cfg.method not in entry.methods:
            _fail(kv["method"][1], f"model '{cfg.model}' does not support method '{cfg.method}' "
                                   f"(supported: {', '.join(entry.methods)})")
    else:
        cfg.method = entry.methods[0]

    dlo, dhi, dplo, dphi, dt1, dh = entry.default_problem(dim, cfg.params)
    cfg.initial_lower = (_resolve_box_side(kv["initial.lower"], "initial.lower", dim, cfg.model, "dimension")
                         if "initial.lower" in kv else [float(v) for v in dlo])
    cfg.initial_upper = (_resolve_box_side(kv["initial.upper"], "initial.upper", dim, cfg.model, "dimension")
                         if "initial.upper" in kv else [float(v) for v in dhi])
    if input_dim == 0:
        for key in ("input.lower", "input.upper"):
            if key in kv:
                _fail(kv[key][1], f"model '{cfg.model}' takes no inputs")
    else:
        cfg.input_lower = (_resolve_box_side(kv["input.lower"], "input.lower", input_dim, cfg.model,
                                             "input dimension") if "input.lower" in kv else list(dplo))
        cfg.input_upper = (_resolve_box_side(kv["input.upper"], "input.upper", input_dim, cfg.model,
                                             "input dimension") if "input.upper" in kv else list(dphi))

    def dbl(key, default):
        return _parse_double(kv[key][0], key, kv[key][1]) if key in kv else default

    cfg.t0 = dbl("t0", 0.0)
    cfg.t1 = dbl("t1", dt1)
    cfg.h = dbl("h", dh)
    if "tube_stride" in kv:
        cfg.tube_stride = _parse_uint(kv["tube_stride"][0], "tube_stride", kv["tube_stride"][1])
    if "workers" in kv:
        w = _parse_uint(kv["workers"][0], "workers", kv["workers"][1])
        if w > 4096:
            _fail(kv["workers"][1], "workers value is implausibly large")
        cfg.workers = w
    if "epsilon" in kv:
        cfg.epsilon = _parse_double(kv["epsilon"][0], "epsilon", kv["epsilon"][1])
        if not (0.0 < cfg.epsilon < 1.0):
            _fail(kv["epsilon"][1], "epsilon must lie in (0, 1)")
    if "delta" in kv:
        cfg.delta = _parse_double(kv["delta"][0], "delta", kv["delta"][1])
        if not (0.0 < cfg.delta < 1.0):
            _fail(kv["delta"][1], "delta must lie in (0, 1)")
    if "seed" in kv:
        cfg.seed = _parse_uint(kv["seed"][0], "seed", kv["seed"][1])
    if "samples" in kv:
        cfg.samples = _parse_uint(kv["samples"][0], "samples", kv["samples"][1])
    if "output" in kv:
        cfg.output = _trim(kv["output"][0])
        if not cfg.output:
            _fail(kv["output"][1], "empty output path")
    if "format" in kv:
        cfg.format = _trim(kv["format"][0])
        if cfg.format not in ("json", "csv"):
            _fail(kv["format"][1], f"unknown format '{cfg.format}' (expected json or csv)")
    return cfg


def parse_config_file(path: str) -> RunConfig:
    """config.cpp:264-270."""
    try:
        with open(path, "rb") as f:
            text = f.read().decode()
    except OSError:
        raise ValueError("cannot open config file: " + path) from None
    return parse_config(text)


def _fmt(v: float) -> str:
    return "%.17g" % v


def serialize_config(cfg: RunConfig) -> str:
    """config.cpp:272-291 (parse_config(serialize_config(c)) == c)."""
    out = [f"model = {cfg.model}"]
    out += [f"param.{k} = {_fmt(v)}" for k, v in sorted(cfg.params.items())]
    out.append(f"method = {cfg.method}")
    out.append("initial.lower = " + ", ".join(_fmt(v) for v in cfg.initial_lower))
    out.append("initial.upper = " + ", ".join(_fmt(v) for v in cfg.initial_upper))
    if cfg.input_lower:
        out.append("input.lower = " + ", ".join(_fmt(v) for v in cfg.input_lower))
        out.append("input.upper = " + ", ".join(_fmt(v) for v in cfg.input_upper))
    out += [f"t0 = {_fmt(cfg.t0)}", f"t1 = {_fmt(cfg.t1)}", f"h = {_fmt(cfg.h)}",
            f"tube_stride = {cfg.tube_stride}", f"workers = {cfg.workers}",
            f"epsilon = {_fmt(cfg.epsilon)}", f"delta = {_fmt(cfg.delta)}", f"seed = {cfg.seed}",
            f"samples = {cfg.samples}", f"output = {cfg.output}", f"format = {cfg.format}"]
    return "\n".join(out) + "\n"


# ------------------------------------------------------------- GPU routing

@dataclass
class BuiltProblem:
    problem: ReachProblem
    mc: MonteCarloSpec
    method: str


def resolve_workers(requested: int) -> int:
    """driver.cpp:38-41 with GPUs for threads: 0 = one shard lane per visible GPU."""
    if requested > 0:
        return requested
    from . import _lib

    return max(1, int(_lib.lib().pirk_device_count()))


def build_problem(cfg: RunConfig) -> BuiltProblem:
    """driver.cpp:43-60."""
    entry = find_model(cfg.model)
    if entry is None:
        raise ValueError("unknown model: " + cfg.model)
    if entry.make is None:
        raise ValueError(f"model '{cfg.model}' has no device kernel in this library "
                         "(out of the hot-path scope, DESIGN.md)")
    model = entry.make(cfg.params)
    inputs = IntervalVector(cfg.input_lower, cfg.input_upper) if model.input_dim > 0 else None
    problem = ReachProblem(model, IntervalVector(cfg.initial_lower, cfg.initial_upper), inputs, cfg.t0, cfg.t1,
                           cfg.h, cfg.tube_stride)
    validate(problem)
    return BuiltProblem(problem, MonteCarloSpec(cfg.epsilon, cfg.delta, cfg.seed, cfg.samples), cfg.method)


@dataclass
class RunOutputs:
    tube: object
    tube_path: str
    report_path: str


def run_config(cfg: RunConfig, ctx=None) -> RunOutputs:
    """driver.cpp:62-72: build, dispatch on the device, write the tube
    (``<output>.json`` / ``.csv``) and ``<output>.report.json``."""
    from .driver import dispatch, report_to_json, tube_to_json
    from .reach import tube_to_csv

    built = build_problem(cfg)
    workers = resolve_workers(cfg.workers)
    tube = dispatch(built.method, built.problem, built.mc, workers, ctx=ctx)
    parent = os.path.dirname(cfg.output)
    if parent:
        os.makedirs(parent, exist_ok=True)
    tube_path = cfg.output + (".csv" if cfg.format == "csv" else ".json")
    report_path = cfg.output + ".report.json"
    with open(tube_path, "w") as f:
        f.write(tube_to_csv(tube) if cfg.format == "csv" else tube_to_json(tube))
    with open(report_path, "w") as f:
        f.write(report_to_json(tube.report))
    return RunOutputs(tube, tube_path, report_path)
