"""Build the device library libpirk_b200.so in-tree (sm_100a only).

Translation units (see csrc/common.cuh for the arithmetic-mode contract):
  inst_exact.cu  -fmad=false -DPIRK_TU_EXACT=1   bit-exact kernels + epilogues
  inst_fast.cu   -DPIRK_TU_EXACT=0               FMA / restructured kernels
  engine.cu                                      host engine + extern "C" ABI
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libpirk_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-ccbin", "/usr/bin/g++",
          "--expt-relaxed-constexpr"]
UNITS = {
    "inst_exact.cu": ["-fmad=false", "-DPIRK_TU_EXACT=1"],
    "inst_fast.cu": ["-DPIRK_TU_EXACT=0"],
    "engine.cu": [],
}


def _sources():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)
            if f.endswith((".cu", ".cuh", ".h"))] + [
        os.path.join(HERE, "..", "include", "pirk_c.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in _sources())


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile the three translation units and link `out`.  `defines` (extra
    -D flags) and `out` exist for development A/B builds (tools/ab_build.py)."""
    if not force and out == LIB and up_to_date():
        return LIB
    libdir = os.path.dirname(out)
    os.makedirs(libdir, exist_ok=True)
    objdir = os.path.join(libdir, "obj" if out == LIB else "obj_" + os.path.basename(out))
    os.makedirs(objdir, exist_ok=True)

    def compile_one(item):
        src, flags = item
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *COMMON, *flags, *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, src),
               "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return obj, r.stderr

    with ThreadPoolExecutor(max_workers=len(UNITS)) as ex:
        results = list(ex.map(compile_one, UNITS.items()))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    objs = [o for o, _ in results]
    tmp = out + ".tmp"
    # NVRTC compiles user-defined models at run time (csrc/user_models.cuh)
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-ccbin", "/usr/bin/g++", *objs,
           "-lnvrtc", "-Xlinker", "-rpath=/usr/local/cuda/lib64", "-o", tmp]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
