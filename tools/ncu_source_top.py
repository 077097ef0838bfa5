"""Top SASS lines of an `ncu --page source --csv` export by warp-stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for hi, r in enumerate(rows):
    if "Source" in r and "Warp Stall Sampling (All Samples)" in r:
        break
h = rows[hi]
si, ws, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for r in rows[hi + 1:]:
    try:
        data.append((float(r[ws] or 0), float(r[ie] or 0), r[0][-5:], r[si].strip()[:90]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
for d in sorted(data, reverse=True)[:n]:
    print("%5.1f%%  exec=%-9d %s  %s" % (100 * d[0] / tot, d[1], d[2], d[3]))
