"""Summarise an .ncu-rep: headline metrics + SASS opcode mix with stall share."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
det = run("--page", "details", "--csv")
keys = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "L2 Hit Rate", "Warp Cycles Per Issued Instruction",
        "Registers Per Thread", "SM Frequency"]
for r in csv.reader(io.StringIO(det)):
    if len(r) > 3 and r[-3] in keys:
        print(f"{r[-3]:36s} {r[-1]:>12s} {r[-2]}")
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
for name in ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
             "smsp__inst_executed.sum", "launch__grid_size", "launch__registers_per_thread"]:
    if name in h:
        i = h.index(name); print(f"{name:60s} {v[i]:>14s} {u[i]}")
sass = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source=sass"))))
hh = sass[1]; data = sass[2:]
ia = hh.index("Instructions Executed"); isrc = hh.index("Source")
iss = [i for i, x in enumerate(hh) if x.startswith("Warp Stall Sampling (All")][0]
ops = collections.Counter(); st = collections.Counter(); tot = 0
for r in data:
    try: n = int(r[ia])
    except Exception: continue
    t = r[isrc].split()
    op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "?")).split(".")[0]
    ops[op] += n; tot += n
    try: st[op] += int(r[iss])
    except Exception: pass
S = sum(st.values()) or 1
print("total warp instructions", tot)
for op, n in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 16):
    print(f"  {op:10s} {n:13d} {100*n/tot:5.1f}%   stall-samples {100*st[op]/S:5.1f}%")
