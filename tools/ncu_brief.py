"""Headline counters of one ncu report (first launch): time, instructions, issue, tensor pipe, stalls."""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, v = r[0], r[2]
want = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
for w in want:
    if w in h:
        print(f"{w:70s} {v[h.index(w)]}")
print("stalls (warps per issue-active cycle):")
st = []
for i, x in enumerate(h):
    if x.startswith("smsp__average_warps_issue_stalled") and x.endswith("per_issue_active.ratio"):
        try:
            st.append((float(v[i]), x.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
for val, nm in sorted(st, reverse=True)[:9]:
    print(f"  {nm:30s} {val:.2f}")
