"""Per-source-line executed warp instructions of one kernel (ncu source page csv)."""
import csv, gzip, sys, collections
path, pat = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
op = gzip.open if path.endswith(".gz") else open
fn, hdr, per = None, None, collections.Counter()
src = {}
with op(path, "rt") as f:
    for row in csv.reader(f):
        if len(row) >= 2 and row[0] == "Function Name":
            fn = row[1]; continue
        if row and row[0] == "Line No":
            hdr = row; continue
        if fn is None or pat not in fn or hdr is None or len(row) < len(hdr):
            continue
        if not row[0]:  # SASS rows carry no line number in this export
            continue
        try:
            v = int(row[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        per[row[0]] += v
        src[row[0]] = row[1][:100]
tot = sum(per.values())
print("warp instructions", tot)
for ln, v in per.most_common(n):
    print(f"{v:10d} {100.0 * v / max(tot, 1):5.1f}%  {ln:>5}  {src[ln]}")
