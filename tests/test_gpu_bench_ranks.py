"""The N > 1 bench path on one B200: `bench.py --gpus 2` under torchrun with
two ranks on cuda:0 (--same-device, gloo with host-staged halos) at a reduced
grid.  Exercises the sharded device bench (z-slab halos, interior/boundary
split), the sharded e2e call, the sharded C4 chain line and every max-over-ranks
reduction, the sharded Monte Carlo line -- the code the driver's 8-GPU scaling
run executes with NCCL."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_one_gpu():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo", "--same-device",
           "--grid", "256", "--steps", "4", "--warmup", "3", "--no-exact", "--chain-n", "200000"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["check"]["finite_ordered_bounded"] and line["check"]["plane_invariance_ok"]
    assert line["roofline"]["per"] == "step (per rank)" and line["roofline"]["launches_per_step"] >= 1
    e2e = line["e2e"]
    assert e2e["value"] > 0 and not e2e["order_violated"] and e2e["rk4_steps"] == 100
    c4 = line["secondary"]["C4_chain_sharded_nGPU"]
    assert c4["n_gpus"] == 2 and c4["value"] > 0
    c2 = line["secondary"]["C2_mc_sharded_nGPU"]
    assert c2["n_gpus"] == 2 and c2["hull_ok"] and c2["value"] > 0
