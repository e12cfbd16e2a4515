"""Per-kernel summary of ncu CSV exports (scripts/gpu_ncu_all.sh keeps the
--page raw / details CSVs, gzipped, instead of the .ncu-rep files).

    python scripts/ncu_csv_summary.py raw <X_raw.csv.gz>        # one line per captured kernel
    python scripts/ncu_csv_summary.py launches <launches.csv.gz>  # per-kernel totals of a launch list
"""
import collections
import csv
import gzip
import io
import sys

RAW = [("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rdMB"), ("dram__bytes_write.sum", "wrMB"),
       ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM%"),
       ("lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "L2%"),
       ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM%"),
       ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
       ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
       ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"), ("launch__block_size", "block")]


def raw(path):
    rows = list(csv.reader(io.TextIOWrapper(gzip.open(path))))
    hdr, units, data = rows[0], rows[1], rows[2:]
    stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    print("%-28s " % "kernel" + " ".join("%8s" % l for _, l in RAW) + "     GB/s  top stalls (pc samples)")
    for r in data:
        name = r[hdr.index("Kernel Name")].split("(")[0].split("::")[-1]
        vals = []
        for m, _ in RAW:
            if m not in hdr:
                vals.append("-")
                continue
            v = r[hdr.index(m)].replace(",", "")
            u = units[hdr.index(m)]
            try:
                x = float(v)
                if u == "Kbyte":
                    x /= 1e3
                elif u == "byte":
                    x /= 1e6
                elif u == "Gbyte":
                    x *= 1e3
                elif u == "ms" or u == "msecond":
                    x *= 1e3
                elif u == "ns" or u == "nsecond":
                    x /= 1e3
                vals.append("%8.1f" % x)
            except ValueError:
                vals.append("%8s" % v[:8])
        try:  # achieved DRAM bandwidth of the capture (cold caches): (read + write) / duration
            gbs = "%9.1f" % ((float(vals[1]) + float(vals[2])) * 1e6 / (float(vals[0]) * 1e-6) / 1e9)
        except (ValueError, ZeroDivisionError):
            gbs = "%9s" % "-"
        tot = sum(float(r[i] or 0) for i in stall) or 1.0
        top = sorted(((float(r[i] or 0), hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", "")) for i in stall),
                     reverse=True)[:3]
        print("%-28s " % name[:28] + " ".join(vals) + gbs + "  " + " ".join("%s %.0f%%" % (n, 100 * v / tot) for v, n in top))


def launches(path):
    rows = list(csv.reader(io.TextIOWrapper(gzip.open(path))))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1,
             "msecond": 1e3, "ms": 1e3}
    by = collections.defaultdict(dict)
    for d in data:
        by[(int(d["ID"]), d["Kernel Name"].split("(")[0].split("::")[-1])][d["Metric Name"]] = \
            float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, n), v in by.items():
        a = agg[n]
        a[0] += 1
        a[1] += v.get("gpu__time_duration.sum", 0.0)
        a[2] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
    T = sum(a[1] for a in agg.values())
    B = sum(a[2] for a in agg.values())
    print("launches %d, serialised kernel time %.2f ms, DRAM %.3f GB" % (len(by), T / 1e3, B / 1e9))
    print("%-40s %6s %10s %7s %10s %10s" % ("kernel", "n", "time_us", "share", "dram_MB", "MB/launch"))
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print("%-40s %6d %10.1f %6.1f%% %10.1f %10.3f" % (n[:40], a[0], a[1], 100 * a[1] / T, a[2] / 1e6, a[2] / 1e6 / a[0]))


if __name__ == "__main__":
    {"raw": raw, "launches": launches}[sys.argv[1]](sys.argv[2])
