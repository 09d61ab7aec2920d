"""Summarise an ncu --metrics gpu__time_duration.sum CSV: per-kernel totals over one step."""
import csv, collections, sys
path = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
count = int(sys.argv[3]) if len(sys.argv) > 3 else 10**9
lines = open(path).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = [r for r in csv.DictReader(lines[start:]) if r['Metric Name'] == 'gpu__time_duration.sum']
rows = [r for r in rows if 'smpk' in r['Kernel Name']]
rows = rows[skip:skip + count]
agg = collections.OrderedDict()
tot = 0.0
for r in rows:
    k = (r['Kernel Name'].split('(')[0][:48], r['Grid Size'])
    t = float(r['Metric Value']) / 1e3
    a = agg.setdefault(k, [0, 0.0]); a[0] += 1; a[1] += t; tot += t
print(f"{len(rows)} launches, total {tot:.1f} us")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:9.1f} us {100*t/tot:5.1f}% {n:4d}x {t/n:8.1f} us/launch  {k[0]} grid={k[1]}")
