"""Summarise an ncu csv with gpu__time_duration.sum + dram bytes per launch:
per kernel name: count, total us, DRAM GB read/written, achieved DRAM GB/s."""
import csv, sys, collections
path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii, ui = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('ID'), hdr.index('Metric Unit')
launch = collections.OrderedDict()
for r in rows[1:]:
    d = launch.setdefault(r[ii], {"name": r[ki]})
    v = float(r[vi].replace(',', ''))
    u = r[ui]
    if 'time' in r[mi]:
        v *= {'ns': 1e-3, 'us': 1.0, 'ms': 1e3, 's': 1e6}.get(u, 1.0)
    else:
        v *= {'byte': 1.0, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'Tbyte': 1e12}.get(u, 1.0)
    d[r[mi]] = v
items = list(launch.values())
if len(sys.argv) > 2:
    items = items[-int(sys.argv[2]):]
agg = collections.OrderedDict()
for d in items:
    key = d["name"].split('(')[0][-56:]
    a = agg.setdefault(key, [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get('gpu__time_duration.sum', 0.0)
    a[2] += d.get('dram__bytes_read.sum', 0.0)
    a[3] += d.get('dram__bytes_write.sum', 0.0)
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    bw = (a[2] + a[3]) / a[1] / 1e3 if a[1] else 0.0
    print(f"{a[1]:12.1f} us {100*a[1]/tot:5.1f}% x{a[0]:<4d} rd {a[2]/1e9:9.3f} GB wr {a[3]/1e9:9.3f} GB {bw:7.0f} GB/s  {k}")
print(f"{tot:12.1f} us total, {len(items)} launches")
