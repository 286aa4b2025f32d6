"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (second half = timed solve)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]; data = rows[hdr_i + 1:]
ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
part = data[len(data) // 2:] if len(sys.argv) < 3 else data
agg = collections.OrderedDict()
for r in part:
    name = r[ki].split('(')[0][:56]
    a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += float(r[vi].replace(',', ''))
tot = sum(v[1] for v in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
    print(f"{k:56s} {c:4d} {t/1e6:9.3f} ms {100*t/tot:5.1f}%")
print(f"total {tot/1e6:.3f} ms, {len(part)} launches")
