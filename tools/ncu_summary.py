#!/usr/bin/env python3
"""Summarise an ncu --set full report (.ncu-rep) into JSON for profiles/.

usage: tools/ncu_summary.py REPORT.ncu-rep OUT.json [--alg-bytes N]
Reads `ncu -i --page raw --csv`; records per-launch duration, DRAM bytes (the roofline
`traffic`), throughput percentages, occupancy, registers and the top warp-stall reasons.
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def main():
    rep, out = sys.argv[1], sys.argv[2]
    alg = None
    if "--alg-bytes" in sys.argv:
        alg = float(sys.argv[sys.argv.index("--alg-bytes") + 1])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for v in rows[2:]:
        d = {"kernel": v[hdr.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{v[i]} {units[i]}".strip()
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(v[i]), h.split("stalled_")[1].split("_per_issue")[0]))
                except ValueError:
                    pass
        d["top_stalls_per_issue"] = [[n, round(x, 3)] for x, n in sorted(stalls, reverse=True)[:6]]
        launches.append(d)

    def num(s, scale):
        x, u = s.split()[0], (s.split()[1] if len(s.split()) > 1 else "")
        f = float(x)
        return f * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(u, 1) if scale else f

    first = launches[0]
    rd = num(first["dram__bytes_read.sum"], True)
    wr = num(first["dram__bytes_write.sum"], True)
    summary = {"report": rep, "launches": launches, "dram_bytes_per_launch": rd + wr}
    if alg:
        summary["algorithmic_bytes_per_launch"] = alg
        summary["traffic_over_algorithmic"] = (rd + wr) / alg
    with open(out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
