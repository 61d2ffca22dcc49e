"""Tube / report / bench serialisations against golden files written by the
reference's own io.cpp and driver.cpp (oracle/ref_io_golden.cpp; fixtures in
tests/golden/io/).  CPU-only: tubes come from the oracle restatement, which is
bit-identical to the reference (tests/test_oracle.py); the GPU-side check is
test_gpu_parity.py::test_tube_formats_match_reference_io."""
import json
import os

import numpy as np
import pytest

import paper_2001_10635_b200 as pk
from paper_2001_10635_b200 import driver as D
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return f.read()


def report_from(obj):
    ph = obj["phases"]
    return pk.RunReport(method=obj["method"], n=obj["n"], m=obj["m"], workers=obj["workers"],
                        steps=obj["steps"], peak_state_bytes=obj["peak_state_bytes"],
                        phases=pk.PhaseTimes(ph["setup_s"], ph["integration_s"], ph["reduction_s"]))


def tube_from(method, times, lower, upper, report):
    entries = [pk.TubeEntry(float(t), pk.IntervalVector(lo, hi)) for t, lo, hi in zip(times, lower, upper)]
    return pk.ReachTube(method, entries, report)


def test_synthetic_json_matches_nlohmann():
    """Double formatting corner cases (tiny, huge, 1e15 <= |v| < 1e16, 5e-324)."""
    lo = [[-1e-05, 1.0, 123456789.0, -0.1], [-3.0, 1.0 / 3.0, 5e-324, 1e15]]
    hi = [[1e-300, 1e+20, 1.2345678901234567e+16, 2.5], [-2.0, 2.0 / 3.0, 1e-4, 1e16]]
    rep = pk.RunReport(method="monte-carlo", n=4, m=1000, workers=3, steps=7, peak_state_bytes=123456,
                       phases=pk.PhaseTimes(1.5e-06, 2.0, 0.0))
    tube = tube_from("monte-carlo", [0.0, 0.1], lo, hi, rep)
    assert D.tube_to_json(tube) == gold("synthetic.json")
    assert D.report_to_json(rep) == gold("synthetic.report.json")


def test_bench_csv_matches_reference():
    rows = [D.BenchRow(1000, 1, 0.0123456789, 60, "ok"), D.BenchRow(1000, 8, 0.5, 60, "ok"),
            D.BenchRow(64, 2, 0.0, 0, "error: bad, input")]
    assert D.bench_csv(rows) == gold("bench.csv")


def test_traffic_tube_csv_json_match_reference():
    """ivreach::mixed_monotonicity(traffic n=5) through io.cpp vs the oracle's
    tube through our formatters: byte-identical."""
    m = pk.make_traffic(5)
    ref = O.mixed_monotonicity(m, 10.0, 20.0, 4.0, 6.0, 0.0, 3.0, 0.5, 2)
    rep = report_from(json.loads(gold("traffic_mm.json"))["report"])
    tube = tube_from("mixed-monotonicity", ref.times, ref.lower, ref.upper, rep)
    assert D.tube_to_csv(tube) == gold("traffic_mm.csv")
    assert D.tube_to_json(tube) == gold("traffic_mm.json")


def test_dispatch_rejects_unknown_method():
    with pytest.raises(ValueError, match="unknown method: bogus"):
        D.dispatch("bogus", None)


def test_bench_validates_arguments():
    with pytest.raises(ValueError, match="no dimensions"):
        D.bench("traffic", "mixed-monotonicity", [], [1], 1, 0.0, 1.0, 0.5)
    with pytest.raises(ValueError, match="no worker counts"):
        D.bench("traffic", "mixed-monotonicity", [10], [], 1, 0.0, 1.0, 0.5)
    with pytest.raises(ValueError, match="repetitions"):
        D.bench("traffic", "mixed-monotonicity", [10], [1], 0, 0.0, 1.0, 0.5)
    with pytest.raises(ValueError, match="unknown model"):
        D.bench("nope", "mixed-monotonicity", [10], [1], 1, 0.0, 1.0, 0.5)


def test_bench_turns_failures_into_rows():
    """A problem the validator rejects (h <= 0) becomes an error row, as in
    driver.cpp:97-103, without touching the device."""
    rows = D.bench("traffic", "mixed-monotonicity", [10], [1, 2], 1, 0.0, 1.0, -0.5)
    assert [r.status.startswith("error: ") for r in rows] == [True, True]
    assert [r.workers for r in rows] == [1, 2]
    assert D.bench_csv(rows).splitlines()[1].startswith("10,1,,0,error: ")
