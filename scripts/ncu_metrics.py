"""Print the key --set full metrics of every kernel in an ncu report.

usage: python scripts/ncu_metrics.py report.ncu-rep [extra-substring ...]
"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Executed Ipc Active",
        "Compute (SM) Throughput", "DRAM Throughput", "Executed Instructions", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction", "Block Limit Registers",
        "Block Limit Shared Mem"] + sys.argv[2:]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = {k: i for i, k in enumerate(rows[0])}
cur = None
for r in rows[1:]:
    name = (r[h["ID"]], r[h["Kernel Name"]])
    if name != cur:
        cur = name
        print("==", name[0], name[1][:90])
    if r[h["Metric Name"]] in KEYS:
        print(f"   {r[h['Metric Name']]:40s} {r[h['Metric Value']]:>14s} {r[h['Metric Unit']]}")
