"""Config files through the GPU path: each shipped
reference config (its resolved form, tests/golden/io/configs/<name>.parsed)
runs through paper_2001_10635_b200.config.run_config on the device and must
write the tube the reference's run_config wrote (oracle/_ref, same file):
boxes bit-identical in exact mode (arch-quadrotor: CUDA vs glibc trig, 1e-12),
report fields identical except wall-clock phases."""
import json
import os

import numpy as np
import pytest

import paper_2001_10635_b200 as pk
from paper_2001_10635_b200 import config as CF

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io", "configs")
RUNNABLE = ["traffic", "heat3d", "laub-loomis", "arch-quadrotor", "vdp", "vdp-mc", "scalar-decay",
            "scalar-linear"]


@pytest.mark.parametrize("name", RUNNABLE)
def test_run_config_writes_the_reference_tube(name, tmp_path):
    cfg = CF.parse_config(open(os.path.join(GOLD, name + ".parsed")).read())
    cfg.output = str(tmp_path / "out" / name)
    cfg.workers = 1
    pk.set_default_mode("exact")
    out = CF.run_config(cfg)
    got = json.load(open(out.tube_path))
    want = json.load(open(os.path.join(GOLD, name + ".json")))
    assert got["method"] == want["method"] and got["times"] == want["times"]
    lo = np.array([b["lower"] for b in got["boxes"]])
    hi = np.array([b["upper"] for b in got["boxes"]])
    wlo = np.array([b["lower"] for b in want["boxes"]])
    whi = np.array([b["upper"] for b in want["boxes"]])
    if name == "arch-quadrotor":
        assert np.allclose(lo, wlo, rtol=1e-12, atol=1e-14) and np.allclose(hi, whi, rtol=1e-12, atol=1e-14)
    else:
        assert np.array_equal(lo, wlo) and np.array_equal(hi, whi)
    rep = json.load(open(out.report_path))
    wrep = json.load(open(os.path.join(GOLD, name + ".report.json")))
    for k in ("method", "n", "m", "steps", "peak_state_bytes", "workers"):
        assert rep[k] == wrep[k], k


def test_cli_run(tmp_path):
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(GOLD, "vdp.parsed")).read().replace("output = out/vdp",
                                                                  f"output = {tmp_path}/vdp")
    cfgp = tmp_path / "vdp.cfg"
    cfgp.write_text(text)
    r = subprocess.run([sys.executable, "-m", "paper_2001_10635_b200", "run", str(cfgp), "--workers", "1"],
                       cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    got = json.load(open(tmp_path / "vdp.json"))
    want = json.load(open(os.path.join(GOLD, "vdp.json")))
    assert got["boxes"] == want["boxes"]
