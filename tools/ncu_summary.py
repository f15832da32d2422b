"""Summarise an .ncu-rep (details page) into a compact table: python tools/ncu_summary.py rep [names...]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
want = sys.argv[2:] or ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
    "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy",
    "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
    "Avg. Not Predicated Off Threads Per Warp", "Branch Instructions Ratio", "L1/TEX Hit Rate", "L2 Hit Rate",
    "Block Limit Shared Mem", "Block Limit Registers", "Dynamic Shared Memory Per Block", "Static Shared Memory Per Block",
    "Executed Instructions", "Grid Size", "Block Size"]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.DictReader(io.StringIO(out)))
seen = {}
for r in rows:
    k = (r["ID"], r["Kernel Name"].split("(")[0])
    if r["Metric Name"] in want:
        seen.setdefault(k, {})[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
for k, d in seen.items():
    print(f"== launch {k[0]} {k[1]}")
    for m in want:
        if m in d:
            print(f"   {m:45s} {d[m][0]:>14s} {d[m][1]}")
