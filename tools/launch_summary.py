"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per kernel
name, count and total microseconds (last step only when --last N)."""
import csv, sys, collections
path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index('Kernel Name'), hdr.index('Metric Value')
data = [(r[ki], float(r[vi].replace(',', ''))) for r in rows[1:]]
if len(sys.argv) > 2:
    data = data[-int(sys.argv[2]):]
agg = collections.OrderedDict()
for k, v in data:
    key = k.split('(')[0][-60:]
    c, t = agg.get(key, (0, 0.0))
    agg[key] = (c + 1, t + v / 1000.0)
tot = sum(t for _, t in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.1f} us {100*t/tot:5.1f}%  x{c:<4d} {k}")
print(f"{tot:10.1f} us total, {len(data)} launches")
