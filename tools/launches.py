"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; data = rows[hi + 1:]
ki, vi, ii = h.index('Kernel Name'), h.index('Metric Value'), h.index('ID')
seq = [(int(r[ii]), r[ki].split('(')[0].split('::')[-1][:48], float(r[vi].replace(',', ''))) for r in data]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tot = sum(v for _, _, v in seq[-last:])
agg = collections.OrderedDict()
for i, n, v in seq[-last:]:
    agg.setdefault(n, [0, 0.0]); agg[n][0] += 1; agg[n][1] += v
for n, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:50s} x{c:3d} {v/1e3:10.1f} us  {100*v/tot:5.1f}%")
print(f"total {tot/1e3:.1f} us over last {last} launches")
