"""Summarises an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= mi:
        continue
    v = float(r[mi].replace(",", ""))
    v = v / 1e3 if r[ui] in ("ns", "nsecond") else v * 1e3 if r[ui] in ("ms", "msecond") else v
    name = r[ki].replace("(anonymous namespace)::", "")
    m = re.search(r"(k_\w+|cub::\w+)", name)
    key = m.group(1) if m else name[:40]
    a = agg[key]
    a[0] += 1
    a[1] += v
    a[2] = max(a[2], v)
    tot += v
print("%-40s %7s %12s %7s %10s %10s" % ("kernel", "n", "total_us", "share", "avg_us", "max_us"))
for k, (n, t, mx) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%-40s %7d %12.1f %6.1f%% %10.2f %10.2f" % (k, n, t, 100 * t / tot, t / n, mx))
print("total kernel time %.3f ms over %d launches" % (tot / 1e3, sum(a[0] for a in agg.values())))
