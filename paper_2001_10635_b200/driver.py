"""Driver-level wiring of the reach entry points:
method dispatch, the dimension x worker bench sweep, and the reference's tube /
report serialisations, byte-compatible with ivreach's io.cpp.

* ``dispatch``           driver.cpp:28-34
* ``bench`` / ``bench_csv``  driver.cpp:74-138 / :140-156
* ``tube_to_json``, ``report_to_json``  io.cpp:55-67 / :107-109 (nlohmann
  ``dump(2)``: keys sorted, 2-space indent, shortest round-trip doubles)
* ``tube_to_csv``        io.cpp:84-103 (re-exported from ``reach``)

``workers`` keeps the reference's meaning of "parallel resources": here the
number of GPUs a run may use.  In-process runs use one device (workers are
recorded in the report, as the reference records its thread count); multi-GPU
runs go through :mod:`paper_2001_10635_b200.sharded`, one process per GPU.
"""
from __future__ import annotations

import json
import math
import statistics
import time
from dataclasses import dataclass
from decimal import Decimal
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

from . import models as M
from .reach import (IntervalVector, MonteCarloSpec, ReachProblem, ReachTube, RunReport,
                    growth_bound, mixed_monotonicity, monte_carlo, tube_to_csv, validate)

__all__ = ["dispatch", "BenchRow", "bench", "bench_csv", "tube_to_json", "report_to_json",
           "tube_to_csv", "CATALOG"]


def dispatch(method: str, problem: ReachProblem, mc: MonteCarloSpec = MonteCarloSpec(),
             workers: int = 1, ctx=None) -> ReachTube:
    """driver.cpp:28-34: route a method name to its entry point."""
    if method == "growth-bound":
        return growth_bound(problem, workers, ctx=ctx)
    if method == "mixed-monotonicity":
        return mixed_monotonicity(problem, workers, ctx=ctx)
    if method == "monte-carlo":
        return monte_carlo(problem, mc, workers, ctx=ctx)
    raise ValueError("unknown method: " + method)


# ------------------------------------------------------------ serialisation

def _json_double(v: float) -> str:
    """nlohmann::json's number_float output (detail/conversions/to_chars.hpp
    format_buffer with min_exp = -4, max_exp = 15): the shortest round-trip
    digits d_1..d_k of |v| with the decimal point at position n = k + e,
    written as ``ddd000.0`` (k <= n <= 15), ``dd.dd`` (0 < n <= 15),
    ``0.000dd`` (-4 < n <= 0), else ``d.ddde+XX`` (two-digit minimum
    exponent).  Differs from Python's repr for 1e15 <= |v| < 1e16."""
    v = float(v)
    if not math.isfinite(v):
        return "null"  # nlohmann writes NaN / inf as null
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    if v == 0.0:
        return sign + "0.0"
    t = Decimal(repr(abs(v))).normalize().as_tuple()
    digits = "".join(map(str, t.digits))
    k = len(digits)
    n = k + t.exponent
    if k <= n <= 15:
        return sign + digits + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + digits[:n] + "." + digits[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + digits
    e = n - 1
    mant = digits if k == 1 else digits[0] + "." + digits[1:]
    return f"{sign}{mant}e{'-' if e < 0 else '+'}{abs(e):02d}"


def _dump(obj, indent: int = 2, level: int = 0) -> str:
    pad, inner = " " * (indent * level), " " * (indent * (level + 1))
    if isinstance(obj, dict):
        if not obj:
            return "{}"
        items = [f'{inner}{json.dumps(k)}: {_dump(obj[k], indent, level + 1)}' for k in sorted(obj)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(obj, (list, tuple)):
        if not len(obj):
            return "[]"
        return "[\n" + ",\n".join(inner + _dump(v, indent, level + 1) for v in obj) + "\n" + pad + "]"
    if isinstance(obj, bool):
        return "true" if obj else "false"
    if isinstance(obj, (int, np.integer)):
        return str(int(obj))
    if isinstance(obj, (float, np.floating)):
        return _json_double(float(obj))
    if isinstance(obj, str):
        return json.dumps(obj)
    raise TypeError(f"cannot serialise {type(obj)}")


def _report_obj(r: RunReport) -> Dict:
    """io.cpp:21-31."""
    return {"method": r.method, "n": int(r.n), "m": int(r.m), "workers": int(r.workers),
            "steps": int(r.steps), "peak_state_bytes": int(r.peak_state_bytes),
            "phases": {"setup_s": float(r.phases.setup_s),
                       "integration_s": float(r.phases.integration_s),
                       "reduction_s": float(r.phases.reduction_s)}}


def report_to_json(report: RunReport) -> str:
    """io.cpp:107-109."""
    return _dump(_report_obj(report)) + "\n"


def tube_to_json(tube: ReachTube) -> str:
    """io.cpp:55-67: {method, times, boxes: [{lower, upper}], report}."""
    obj = {"method": tube.method,
           "times": [float(e.t) for e in tube.entries],
           "boxes": [{"lower": e.box.lower.tolist(), "upper": e.box.upper.tolist()}
                     for e in tube.entries],
           "report": _report_obj(tube.report)}
    return _dump(obj) + "\n"


# ------------------------------------------------------------ bench sweep

@dataclass
class CatalogEntry:
    """The slice of models.cpp's catalogue the sweep needs: a constructor
    from the size parameter, the size parameter for a target dimension
    (models.hpp size_param_for_dim) and the default problem boxes."""

    make: Callable[[int], M.SystemModel]
    size_for_dim: Callable[[int], int]
    default_boxes: Callable[[M.SystemModel], tuple]


def _traffic_boxes(m):
    return IntervalVector(np.full(m.dim, 10.0), np.full(m.dim, 20.0)), IntervalVector([4.0], [6.0])


def _heat_boxes(m):  # models.cpp:744-745: [0.9, 1.1] broadcast
    return IntervalVector(np.full(m.dim, 0.9), np.full(m.dim, 1.1)), None


def _chain_boxes(m):
    c = np.zeros(m.dim)
    return IntervalVector(c - 0.05, c + 0.05), IntervalVector([-0.1], [0.1])


CATALOG: Dict[str, CatalogEntry] = {
    "traffic": CatalogEntry(M.make_traffic, lambda d: max(1, d), _traffic_boxes),
    "heat3d": CatalogEntry(M.make_heat3d, lambda d: max(2, round(d ** (1.0 / 3.0))), _heat_boxes),
    "chain": CatalogEntry(M.make_chain, lambda d: max(1, d), _chain_boxes),
}


@dataclass
class BenchRow:
    """driver.hpp:33-39."""

    n: int = 0
    workers: int = 1
    median_seconds: float = 0.0
    steps: int = 0
    status: str = "ok"


def bench(model: str, method: str, dims: Sequence[int], workers_list: Sequence[int], reps: int,
          t0: float, t1: float, h: float, tube_stride: int = 0,
          mc: MonteCarloSpec = MonteCarloSpec(), ctx=None) -> List[BenchRow]:
    """driver.cpp:74-138: for each dimension rebuild the model through its
    size parameter with the default boxes, run ``reps`` timed repetitions per
    worker count and report the median; failures become status rows."""
    if not dims:
        raise ValueError("bench: no dimensions given")
    if not workers_list:
        raise ValueError("bench: no worker counts given")
    if reps <= 0:
        raise ValueError("bench: repetitions must be positive")
    entry = CATALOG.get(model)
    if entry is None:
        raise ValueError("unknown model: " + model)
    rows: List[BenchRow] = []
    for dim in dims:
        problem: Optional[ReachProblem] = None
        build_error = ""
        try:
            m = entry.make(entry.size_for_dim(int(dim)))
            init, inputs = entry.default_boxes(m)
            problem = ReachProblem(m, init, inputs, t0, t1, h, tube_stride)
            validate(problem)
        except MemoryError:
            build_error = "oom"
        except Exception as e:  # noqa: BLE001 -- the reference turns every failure into a row
            build_error = "error: " + str(e)
        from .reach import plan_steps
        planned = plan_steps(t0, t1, h).total() if not build_error else 0
        for workers in workers_list:
            row = BenchRow(n=problem.model.dim if problem is not None else int(dim),
                           workers=max(1, int(workers)), steps=planned)
            if build_error:
                row.status = build_error
                rows.append(row)
                continue
            seconds = []
            try:
                for _ in range(reps):
                    t = time.perf_counter()
                    tube = dispatch(method, problem, mc, row.workers, ctx=ctx)
                    seconds.append(time.perf_counter() - t)
                    row.steps = tube.report.steps
                row.median_seconds = statistics.median(seconds)
            except MemoryError:
                row.status = "oom"
            except Exception as e:  # noqa: BLE001
                row.status = "error: " + str(e)
            rows.append(row)
    return rows


def bench_csv(rows: Sequence[BenchRow]) -> str:
    """driver.cpp:140-156: ``n,workers,median_seconds,steps,status``."""
    out = ["n,workers,median_seconds,steps,status"]
    for r in rows:
        med = "%.6f" % r.median_seconds if r.status == "ok" else ""
        out.append(f"{r.n},{r.workers},{med},{r.steps},{r.status.replace(',', ';')}")
    return "\n".join(out) + "\n"
