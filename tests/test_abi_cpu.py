"""CPU: the C-ABI library loads, exports exactly what include/pirk_c.h
declares, and its host-side logic (step planning, record schedule, sample
count, capability table, validation) matches the reference/oracle.  No
compute calls: there is no GPU here, and the library must say so loudly."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2001_10635_b200 as pk
from oracle import oracle as O
from paper_2001_10635_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "pirk_c.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pirk_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), f"{s} missing from libpirk_b200.so"
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table out of sync with pirk_c.h"
    assert L.pirk_abi_version() == 1


def test_library_is_sm100a_only():
    # the product library carries sm_100a SASS (no PTX JIT fallback for other archs)
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_no_gpu_is_an_error_not_a_fallback():
    h = C.c_void_p()
    st = _lib.lib().pirk_create(0, C.byref(h))
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert st == _lib.ECUDA
        with pytest.raises(RuntimeError):
            pk.Context(0)


@pytest.mark.parametrize("t0,t1,h", [(0.0, 30.0, 0.3), (0.0, 1.0, 0.3), (0.0, 0.1, 0.5),
                                     (0.0, 30.0, 0.5), (0.0, 5e-6, 5e-8), (1.5, 2.25, 0.01)])
def test_plan_and_schedule_match_oracle(t0, t1, h):
    p = pk.plan_steps(t0, t1, h)
    assert (p.full_steps, p.has_remainder) == O.plan_steps(t0, t1, h)
    for stride in (0, 1, 3, 10, 1000):
        s1, t1_ = pk.record_schedule(t0, t1, h, stride)
        s2, t2_ = O.record_schedule(t0, t1, h, stride)
        assert np.array_equal(s1, s2) and np.array_equal(t1_, t2_)


def test_sample_count_matches_reference():
    for args in [(2, 0.05, 0.01), (1, 0.5, 0.5), (1, 0.05, 0.01), (12, 0.05, 0.01), (7, 0.01, 1e-6)]:
        assert pk.sample_count(*args) == O.sample_count(*args)
    with pytest.raises(ValueError):
        pk.sample_count(1, 0.0, 0.5)
    with pytest.raises(ValueError):
        pk.sample_count(0, 0.5, 0.5)


def test_capability_table():
    L = _lib.lib()
    sup = lambda m, meth: L.pirk_supports(C.byref(pk.reach.model_struct(m)), meth)
    assert sup(pk.make_traffic(10 ** 6), 0) and sup(pk.make_traffic(10 ** 6), 1)
    assert sup(pk.make_heat3d(1600), 0) and sup(pk.make_heat3d(1600), 1)
    assert sup(pk.make_chain(10 ** 7), 0) and not sup(pk.make_chain(10 ** 7), 1)
    assert not sup(pk.make_arch_quadrotor(), 0)
    assert sup(pk.with_jacobian_decomposition(pk.make_arch_quadrotor()), 0)
    assert sup(pk.make_arch_quadrotor(), 1) and sup(pk.make_arch_quadrotor(), 2)
    # MC: compiled kernels for n <= 64, generated-source (NVRTC) kernel for n <= 1024
    assert sup(pk.make_traffic(100), 2) and sup(pk.make_heat3d(10), 2)
    assert not sup(pk.make_traffic(2000), 2) and not sup(pk.make_heat3d(11), 2)


def test_interval_and_problem_validation_messages():
    # interval.cpp:10-23 / system_model.cpp:10-32
    with pytest.raises(ValueError, match="lower > upper at component 1"):
        pk.IntervalVector([0.0, 2.0], [1.0, 1.0])
    with pytest.raises(ValueError, match="non-finite bound at component 0"):
        pk.IntervalVector([np.nan], [1.0])
    with pytest.raises(ValueError, match="dimension must be at least 1"):
        pk.IntervalVector([], [])
    m = pk.make_traffic(5)
    box = pk.IntervalVector(np.zeros(5), np.ones(5))
    with pytest.raises(ValueError, match="1 inputs but no input box"):
        pk.validate(pk.ReachProblem(m, box, None, 0.0, 1.0, 0.1))
    with pytest.raises(ValueError, match="t0 must be earlier"):
        pk.validate(pk.ReachProblem(m, box, pk.IntervalVector([0.0], [1.0]), 1.0, 1.0, 0.1))
    with pytest.raises(ValueError, match="step size h must be positive"):
        pk.validate(pk.ReachProblem(m, box, pk.IntervalVector([0.0], [1.0]), 0.0, 1.0, 0.0))
    with pytest.raises(ValueError, match="no inputs but an input box"):
        pk.validate(pk.ReachProblem(pk.make_zero(5), box, pk.IntervalVector([0.0], [1.0]), 0.0,
                                    1.0, 0.1))


def test_model_constructor_validation():
    # models.cpp require() messages
    with pytest.raises(ValueError, match="at least 3 segments"):
        pk.make_traffic(2)
    with pytest.raises(ValueError, match="beta must lie in"):
        pk.make_traffic(5, beta=1.5)
    with pytest.raises(ValueError, match="at least 2 grid points"):
        pk.make_heat3d(1)
    with pytest.raises(ValueError, match="jacobian decomposition"):
        pk.with_jacobian_decomposition(pk.make_traffic(5))


def test_interval_helpers():
    b = pk.IntervalVector([0.0, 1.0], [2.0, 5.0])
    assert np.array_equal(pk.center(b), [1.0, 3.0])
    assert np.array_equal(pk.half_width(b), [1.0, 2.0])
    assert pk.from_center_radius([1.0, 3.0], [1.0, 2.0]) == b
    assert pk.contains(b, [2.0, 1.0]) and not pk.contains(b, [2.1, 1.0])
    assert pk.subset_of(pk.IntervalVector([0.5, 1.0], [1.0, 2.0]), b)
    with pytest.raises(ValueError, match="negative radius"):
        pk.from_center_radius([0.0], [-1.0])


def test_tube_csv_format():
    # io.cpp:84-103: header t,lower0,upper0,... and %.17g values
    tube = pk.ReachTube("mixed-monotonicity",
                        [pk.TubeEntry(0.1, pk.IntervalVector([1.0 / 3.0, -0.0], [2.0, 1e-300]))],
                        pk.RunReport())
    csv = pk.tube_to_csv(tube)
    assert csv == "t,lower0,upper0,lower1,upper1\n0.10000000000000001,0.33333333333333331,2,-0,1e-300\n"
