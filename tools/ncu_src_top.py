"""Top stalled SASS lines of an ncu source-page CSV (ncu -i R --page source --csv --print-source sass)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
isrc = hdr.index("Source")
iss = hdr.index("Warp Stall Sampling (All Samples)")
ie = hdr.index("Instructions Executed")
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
ci = [hdr.index(c) for c in cols]
tot = sum(int(r[iss]) for r in data)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for i in sorted(range(len(data)), key=lambda i: -int(data[i][iss]))[:n]:
    r = data[i]
    top = max(zip(cols, ci), key=lambda z: int(r[z[1]] or 0))[0]
    print(f"{i:5d} {int(r[iss]) / tot * 100:5.1f}% ex={r[ie]:>9} {top:22s} {r[isrc].strip()[:80]}")
