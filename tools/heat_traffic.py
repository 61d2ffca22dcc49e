"""Measure the heat kernel's DRAM bytes per launch at the bench size (GPU box).

Runs one ncu metrics pass (dram__bytes_read/write, one steady-state launch)
per mode over tools/prof_target.py and writes profiles/heat_traffic.json,
which bench.py reports as roofline.traffic.  Usage:
    python tools/heat_traffic.py [grid=1600]
"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
grid = int(sys.argv[1]) if len(sys.argv) > 1 else 1600
out = {}
for mode in ("fast", "exact"):
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "-k", "regex:heat", "-s", "1", "-c", "1", sys.executable,
           os.path.join(ROOT, "tools", "prof_target.py"), "heat", str(grid), mode, "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    txt = r.stdout + r.stderr
    kern = re.search(r"void (heat\w*kernel)<", txt)

    def metric(name):
        m = re.search(name + r"\s+(\w+)\s+([\d.,]+)", txt)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(m.group(1), 1)
        return float(m.group(2).replace(",", "")) * scale

    rd, wr = metric("dram__bytes_read.sum"), metric("dram__bytes_write.sum")
    upd = 2.0 * grid ** 3
    out[mode] = {"dram_bytes_per_update": (rd + wr) / upd, "dram_read": rd, "dram_write": wr,
                 "updates_per_launch": upd, "grid": grid,
                 "kernel": kern.group(1) if kern else None,
                 "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum, heat3d g={grid}, "
                           f"{mode}, 1 steady-state launch (tools/heat_traffic.py)"}
    print(mode, out[mode], flush=True)
dst = os.path.join(ROOT, "gpurun_out", "heat_traffic.json")
os.makedirs(os.path.dirname(dst), exist_ok=True)
with open(dst, "w") as f:
    json.dump(out, f, indent=1)
print("wrote", dst)
