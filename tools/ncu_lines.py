"""Per-source-line stall / shared-memory attribution from an .ncu-rep (cuda,sass view)."""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr, agg = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit() or len(r) < len(hdr):
        continue
    if r[2] not in ("", "-"):  # SASS rows carry an address; the cuda line row aggregates them
        continue
    def f(name):
        try:
            return float(r[hdr.index(name)] or 0)
        except (ValueError, IndexError):
            return 0.0
    key = (fname, int(r[0]))
    agg[key] = (f("Warp Stall Sampling (All Samples)"), f("L1 Wavefronts Shared"),
                f("L1 Wavefronts Shared Excessive"), f("Instructions Executed"), r[1].strip()[:80])
tot = sum(v[0] for v in agg.values()) or 1
wtot = sum(v[1] for v in agg.values()) or 1
print(f"{'stall%':>6} {'smem_wf%':>8} {'excess%':>7} {'insts':>12}  line")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*v[0]/tot:6.1f} {100*v[1]/wtot:8.1f} {100*v[2]/wtot:7.1f} {v[3]:12.0f}  {k[0]}:{k[1]} {v[4]}")
