"""Summary of an `ncu --page details --csv` export: a few headline metrics per
captured kernel (the profiles/r*/ncu_full_summary.txt format)."""
import csv
import sys

WANT = ["Memory Throughput", "DRAM Throughput", "Duration", "Compute (SM) Throughput",
        "Executed Ipc Active", "L2 Hit Rate", "Issued Warp Per Scheduler", "No Eligible",
        "Eligible Warps Per Scheduler", "Registers Per Thread", "Waves Per SM",
        "Block Limit Shared Mem", "Theoretical Occupancy", "Achieved Occupancy"]
rows = {}
order = []
with open(sys.argv[1]) as f:
    for r in csv.DictReader(f):
        k = (r["ID"], r["Kernel Name"].split("(")[0])
        if k not in rows:
            rows[k] = {}
            order.append(k)
        m = r["Metric Name"]
        if m in WANT and m not in rows[k]:
            rows[k][m] = (r["Metric Value"], r["Metric Unit"])
print(sys.argv[2] if len(sys.argv) > 2 else "ncu --set full summary")
for k in order:
    print(f"\n== {k[0]} {k[1]}")
    for m in WANT:
        if m in rows[k]:
            v, u = rows[k][m]
            print(f"  {m:<36} {v} {u}")
