#!/usr/bin/env python
"""Key ncu metrics of a report (details page) as `name = value unit` lines."""
import csv
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active", "Issue Slots Busy",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp", "Executed Instructions",
        "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Active Warps Per SM",
        "L1/TEX Hit Rate", "L2 Hit Rate", "Grid Size", "Compute (SM) Throughput", "SM Frequency",
        "Elapsed Cycles", "Branch Efficiency"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
seen = set()
for r in rows[1:]:
    d = dict(zip(h, r))
    n = d.get("Metric Name")
    if n in WANT and n not in seen:
        seen.add(n)
        print(f"{n} = {d.get('Metric Value')} {d.get('Metric Unit')}")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
if len(rr) >= 3:
    hh, units, vals = rr[0], rr[1], rr[2]
    for key in ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_sector_hit_rate.pct",
                "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]:
        if key in hh:
            i = hh.index(key)
            print(f"{key} = {vals[i]} {units[i]}")
