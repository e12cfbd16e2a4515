"""Per-kernel time and DRAM traffic from an ncu launch list
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum).

  python scripts/traffic.py launches.csv WINDOWS [out.json]

Writes {bytes_per_window, source, per_kernel{...}} for bench.py's roofline
"traffic" (per window = totals / WINDOWS; every window in the capture is the
same C1 solve)."""
import collections
import csv
import json
import re
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1,
        "ms": 1e3, "msecond": 1e3}
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, ni, mi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
idi = h.index("ID")
per = collections.defaultdict(lambda: collections.defaultdict(float))
launch = {}
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    v = float(r[mi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    name = r[ki].replace("(anonymous namespace)::", "")
    m = re.search(r"(k_\w+|cub::\w+)", name)
    key = m.group(1) if m else name[:40]
    launch[r[idi]] = key
    per[key][r[ni]] += v
    per[key]["launch_ids"] += 0
counts = collections.Counter(launch.values())
W = float(sys.argv[2])
tot_t = sum(d["gpu__time_duration.sum"] for d in per.values())
tot_b = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in per.values())
print("%-36s %6s %10s %6s %12s %12s" % ("kernel", "n", "time_us", "share", "dram_MB", "MB/launch"))
for k, d in sorted(per.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    b = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    print("%-36s %6d %10.1f %5.1f%% %12.2f %12.4f" % (k, counts[k], d["gpu__time_duration.sum"],
                                                   100 * d["gpu__time_duration.sum"] / tot_t, b / 1e6,
                                                   b / 1e6 / max(1, counts[k])))
print("per window: %.2f ms kernel time, %.1f MB DRAM" % (tot_t / W / 1e3, tot_b / W / 1e6))
if len(sys.argv) > 3:
    json.dump({"bytes_per_window": int(tot_b / W), "kernel_us_per_window": tot_t / W,
               "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over %g C1 windows (%s); ncu flushes caches before each kernel, so this over-counts live traffic"
                         % (W, sys.argv[1].split("/")[-1]),
               "per_kernel": {k: {"launches": counts[k], "time_us": d["gpu__time_duration.sum"],
                                  "dram_bytes": d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]}
                              for k, d in per.items()}}, open(sys.argv[3], "w"), indent=1)
