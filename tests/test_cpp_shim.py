"""The C++ drop-in shim (include/pirk/ivreach_gpu.hpp): reference-style call
sites compile against it (CPU) and produce the reference's results (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "shim_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2001_10635_b200", "lib")


def build(tmp_path):
    exe = str(tmp_path / "shim_dropin")
    r = subprocess.run(["/usr/bin/g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                        SRC, "-L", LIBDIR, "-lpirk_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_shim_compiles_and_links(tmp_path):
    build(tmp_path)


@pytest.mark.gpu
def test_shim_runs_reference_call_sites(tmp_path):
    exe = build(tmp_path)
    golden = os.path.join(ROOT, "tests", "golden", "io", "traffic_mm.csv")
    r = subprocess.run([exe, golden], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout
