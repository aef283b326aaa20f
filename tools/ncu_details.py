"""Print the headline metrics of an `ncu --page details --csv` export, one
kernel launch per block (used for the ws / v6 comparisons in profiles/)."""
import csv
import sys

WANT = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Registers Per Thread", "Achieved Occupancy",
        "Issue Slots Busy", "No Eligible", "L2 Hit Rate", "Mem Busy", "Max Bandwidth", "Warp Cycles Per Issued Instruction",
        "Executed Ipc Active", "Dynamic Shared Memory Per Block", "Grid Size", "SM Frequency", "Block Size",
        "L1/TEX Hit Rate", "Mem Pipes Busy"]
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    ix = {h: i for i, h in enumerate(rows[0])}
    print("==", f)
    last = None
    for r in rows[1:]:
        if len(r) <= ix["Metric Value"]:
            continue
        if r[ix["Metric Name"]] in WANT:
            key = (r[ix["ID"]], r[ix["Kernel Name"]])
            if key != last:
                print(" --", key[0], key[1][:60])
                last = key
            print(f"    {r[ix['Section Name']][:26]:26s} {r[ix['Metric Name']]:38s} {r[ix['Metric Value']]:>12s} {r[ix['Metric Unit']]}")
