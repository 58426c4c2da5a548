"""Top warp-stall source lines of one kernel in an ncu --page source --csv export."""
import csv, gzip, sys
path, pat = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
op = gzip.open if path.endswith(".gz") else open
fn, rows = None, []
with op(path, "rt") as f:
    for row in csv.reader(f):
        if len(row) >= 2 and row[0] == "Function Name":
            fn = row[1]
            continue
        if len(row) < 6 or row[0] in ("File Path", "Line No") or fn is None or pat not in fn:
            continue
        try:
            s = int(row[4] or 0)
        except ValueError:
            continue
        rows.append((s, row[0], (row[1] or row[3])[:110]))
tot = sum(r[0] for r in rows)
print("samples", tot)
for s, ln, src in sorted(rows, reverse=True)[:n]:
    print(f"{s:7d} {100.0 * s / max(tot, 1):5.1f}%  {ln:>5}  {src}")
