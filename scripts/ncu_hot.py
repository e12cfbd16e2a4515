"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, res = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit() and len(r) > 4 and r[2] == "-":
        try:
            res.append((float(r[4] or 0), float(r[5] or 0), fname, int(r[0]), r[1]))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
print("total samples %d" % tot)
for v, ni, f, ln, src in sorted(res, reverse=True)[:top]:
    print("%6.2f%% (not-issued %5.1f%%) %s:%d | %s" % (100 * v / tot, 100 * ni / tot, f, ln, src.strip()[:90]))
