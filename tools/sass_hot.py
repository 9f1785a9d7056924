"""Top SASS lines of one kernel from `ncu --page source --csv` (stall samples)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia, isrc, iss, iex = (h.index("Address"), h.index("Source"),
                      h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"))
data = [(int(r[iss] or 0), int(r[iex] or 0), r[isrc].strip(), i) for i, r in enumerate(rows[2:]) if len(r) > iex and r[iss].isdigit()]
tot = sum(d[0] for d in data)
totx = sum(d[1] for d in data)
print("total samples", tot, "instructions executed", totx)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for s, x, src, i in sorted(data, key=lambda d: -d[0])[:n]:
    print(f"{i:5d} {s:7d} {100 * s / tot:5.1f}% {x:9d}  {src}")
