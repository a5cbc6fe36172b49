"""Summarise an ncu --set full report of the step kernel into profiles/ (markdown + json).

    python tools/ncu_summary.py gpurun_out/prof_int8_v1.ncu-rep profiles/r1_int8_v1
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_shared_mem",
    "sm__cycles_elapsed.avg",
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep, outbase = sys.argv[1], sys.argv[2]
    hdr, units, data = raw(rep)
    res = {"report": rep, "launches": []}
    for vals in data:
        d = {}
        for i, h in enumerate(hdr):
            if h in KEYS or (h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")):
                try:
                    d[h] = [float(vals[i].replace(",", "")), units[i]]
                except ValueError:
                    d[h] = [vals[i], units[i]]
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        d["kernel"] = name
        res["launches"].append(d)
    json.dump(res, open(outbase + ".json", "w"), indent=1)
    with open(outbase + ".md", "w") as fh:
        for d in res["launches"]:
            fh.write(f"### {d['kernel'][:120]}\n\n| metric | value | unit |\n|---|---|---|\n")
            for k in KEYS:
                if k in d:
                    fh.write(f"| {k} | {d[k][0]} | {d[k][1]} |\n")
            st = sorted(((v[0], k) for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
                         and isinstance(v[0], float)), reverse=True)[:8]
            fh.write("\nTop stall reasons (warps per issue-active cycle):\n\n")
            for v, k in st:
                fh.write(f"- {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}: {v:.2f}\n")
            fh.write("\n")
    print(open(outbase + ".md").read())


if __name__ == "__main__":
    main()
