"""Key raw metrics of an .ncu-rep (smem wavefronts, pipes, stalls, DRAM)."""
import csv, io, re, subprocess, sys

rep = sys.argv[1]
raw = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                 capture_output=True, text=True).stdout)))
h, u, v = raw[0], raw[1], raw[2]
pat = re.compile(r"^(gpu__time_duration.sum|dram__bytes_(read|write).sum|"
                 r"l1tex__data_pipe_lsu_wavefronts_mem_shared(_op_ld|_op_st)?.sum(.pct_of_peak_sustained_elapsed)?|"
                 r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum|local_.*|"
                 r"l1tex__t_bytes_pipe_lsu_mem_local.*sum|smsp__inst_executed.sum|"
                 r"sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active|"
                 r"smsp__issue_active.avg.pct_of_peak_sustained_active|"
                 r"launch__registers_per_thread|sm__warps_active.avg.pct_of_peak_sustained_active|"
                 r"smsp__pcsamp_warps_issue_stalled_[a-z_]+(?<!_not_issued))$")
rows = [(h[i], v[i], u[i]) for i in range(len(h)) if pat.match(h[i])]
stalls = [(n, float(x)) for n, x, _ in rows if "pcsamp" in n and x not in ("", "n/a")]
tot = sum(x for _, x in stalls) or 1.0
for n, x, un in rows:
    if "pcsamp" in n:
        continue
    print(f"{n:70s} {x:>18s} {un}")
print("stall samples (share):")
for n, x in sorted(stalls, key=lambda t: -t[1])[:10]:
    print(f"  {n.replace('smsp__pcsamp_warps_issue_stalled_', ''):28s} {100 * x / tot:5.1f}%")
