"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum[,dram__bytes_read.sum,
dram__bytes_write.sum] --csv): per-kernel totals over one step of launches.

usage: python scripts/launch_summary.py launches.csv [skip] [count]
   skip/count select the launches of one step (e.g. skip = warmup_steps * launches_per_step).
ncu's per-launch times are cold-cache and serialised: use the SHARES, not the absolute times.
"""
import collections
import csv
import sys

path = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
count = int(sys.argv[3]) if len(sys.argv) > 3 else 10 ** 9
lines = open(path).read().splitlines()
start = [i for i, ln in enumerate(lines) if ln.startswith('"ID"')][0]
by_id = collections.OrderedDict()
for r in csv.DictReader(lines[start:]):
    d = by_id.setdefault(r["ID"], {"name": r["Kernel Name"], "grid": r["Grid Size"]})
    try:
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    except ValueError:
        pass
launches = list(by_id.values())[skip:skip + count]
agg = collections.OrderedDict()
tot = 0.0
for d in launches:
    k = d["name"].split("(")[0][:70]
    t = d.get("gpu__time_duration.sum", 0.0) / 1e3  # us
    b = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    a = agg.setdefault(k, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += t
    a[2] += b
    tot += t
print(f"{len(launches)} launches, total {tot:.1f} us (ncu serialised, cold cache)")
print(f"{'us':>9} {'share':>6} {'n':>5} {'us/launch':>10} {'DRAM MB/launch':>15}  kernel")
for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:9.1f} {100 * t / tot:5.1f}% {n:5d} {t / n:10.2f} {b / n / 1e6:15.2f}  {k}")
