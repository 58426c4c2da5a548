"""Per-kernel table of one training step from an ncu --metrics CSV
(gpu__time_duration, dram bytes, tensor-pipe %, grid, registers): the kernels
between the last two k_adam launches. Usage: kernel_table.py metrics.csv [hbm_gbs]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
peak = float(sys.argv[2]) if len(sys.argv) > 2 else 6547.5
h = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
H = rows[h]
iI, iK, iM, iV = (H.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
data = collections.OrderedDict()
for r in rows[h + 1:]:
    if len(r) > iV:
        data.setdefault(r[iI], {"k": r[iK]})[r[iM]] = r[iV]
ks = list(data.values())
adam = [i for i, d in enumerate(ks) if "k_adam" in d["k"]]
step = ks[adam[-2] + 1: adam[-1] + 1]
f = lambda d, m: float(d.get(m, "0").replace(",", "") or 0)
print(f"kernels/step {len(step)}; times are ncu's (serialised, cold L2); GB/s vs {peak} measured HBM")
print(f"{'us':>7} {'DRAM MB':>8} {'GB/s':>6} {'%HBM':>5} {'tensor%':>7} {'grid':>6} {'regs':>4}  kernel")
tot = 0.0
for d in step:
    t = f(d, "gpu__time_duration.sum") / 1000
    b = f(d, "dram__bytes_read.sum") + f(d, "dram__bytes_write.sum")
    tp = f(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
    tot += t
    print(f"{t:7.2f} {b / 1e6:8.2f} {b / t / 1e3:6.0f} {100 * b / t / 1e3 / peak:5.1f} {tp:7.2f} "
          f"{d.get('launch__grid_size', ''):>6} {d.get('launch__registers_per_thread', ''):>4}  "
          f"{d['k'].split('(')[0][:70]}")
print(f"sum {tot:.1f} us")
