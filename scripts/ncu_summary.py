"""Key metrics of every kernel in an ncu report (details page)."""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Grid Size", "Block Size",
        "Dynamic Shared Memory Per Block", "Issue Slots Busy", "No Eligible", "Warp Cycles Per Issued Instruction",
        "L2 Hit Rate", "Branch Efficiency"]
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    seen = set()
    print("==", rep.split("/")[-1])
    for r in rows[1:]:
        d = dict(zip(h, r))
        k = (d.get("Kernel Name", "")[:30], d.get("Metric Name"))
        if d.get("Metric Name") in WANT and k not in seen:
            seen.add(k)
            print("  %-40s %s %s" % (d["Metric Name"], d["Metric Value"], d["Metric Unit"]))
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    if len(rr) > 2:
        hh = rr[0]
        for r in rr[2:]:
            d = dict(zip(hh, r))
            print("  dram read %s %s, write %s %s" % (d.get("dram__bytes_read.sum"), rr[1][hh.index("dram__bytes_read.sum")],
                                                   d.get("dram__bytes_write.sum"), rr[1][hh.index("dram__bytes_write.sum")]))
