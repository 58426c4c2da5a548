"""One training step's kernels (between consecutive k_adam launches) from an ncu launch list."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
H = rows[h]; iK = H.index("Kernel Name"); iV = H.index("Metric Value")
data = [(r[iK], float(r[iV].replace(",", ""))) for r in rows[h + 1:] if len(r) > iV and r[iV]]
ends = [i for i, (k, v) in enumerate(data) if "k_adam" in k]
step = data[ends[-2] + 1: ends[-1] + 1]
print("kernels/step", len(step), "sum us %.1f" % (sum(v for k, v in step) / 1000))
agg = collections.Counter(); cnt = collections.Counter()
for k, v in step:
    n = k.split("(")[0][:70]; agg[n] += v / 1000; cnt[n] += 1
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    print(f"{v:8.2f} us  x{cnt[k]:<3d} {k}")
