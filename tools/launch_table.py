"""Summarise an ncu --csv launch list (gpu__time_duration per kernel)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for i, r in enumerate(rows):
    if "Kernel Name" in r:
        hdr = i; break
h = rows[hdr]
iK, iV, iG, iB = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size"), h.index("Block Size")
data = []
for r in rows[hdr + 1:]:
    if len(r) <= iV: continue
    try: v = float(r[iV].replace(",", ""))
    except ValueError: continue
    data.append((r[iK][:70], r[iG], r[iB], v))
tot = sum(d[3] for d in data)
print(f"{len(data)} launches, total {tot/1000:.1f} us")
for n, g, b, v in data: print(f"{v/1000:8.2f} us  {g:>16} {b:>12}  {n}")
