import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Eligible Warps Per Scheduler", "L2 Hit Rate", "L1/TEX Hit Rate", "Grid Size",
        "Theoretical Occupancy", "Avg. Not Predicated Off Threads Per Warp", "Block Limit Shared Mem", "Block Limit Registers"]
cur = None
for r in rows[1:]:
    d = dict(zip(h, r))
    key = (d["ID"], d["Kernel Name"][:60])
    if key != cur:
        cur = key
        print("==", key)
    if d["Metric Name"] in want:
        print("   ", d["Metric Name"].ljust(42), d["Metric Value"], d["Metric Unit"])
