"""Key metrics of every kernel in an ncu report: python tools/ncu_summary.py rep.ncu-rep"""
import csv, io, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Dynamic Shared Memory Per Block", "Executed Instructions", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Grid Size", "Block Size", "Eligible Warps Per Scheduler",
        "No Eligible", "L1/TEX Hit Rate", "L2 Hit Rate"]
cur = None
for r in rows[1:]:
    d = dict(zip(hdr, r))
    k = (d.get("ID"), d.get("Kernel Name", "")[:70])
    if k != cur:
        cur = k
        print("==", k)
    if d.get("Metric Name") in want:
        print(f"   {d['Metric Name']:40s} {d['Metric Value']:>16s} {d['Metric Unit']}")
