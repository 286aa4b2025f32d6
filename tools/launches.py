"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list.
usage: python tools/launches.py launches.csv [all]
Default: the LAST solve only (from the last k_validate_* launch through its k_fill);
'all': every launch in the file."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]; data = rows[hdr_i + 1:]
ki = hdr.index('Kernel Name'); vi = hdr.index('Metric Value')
if len(sys.argv) < 3:
    starts = [i for i, r in enumerate(data) if 'k_validate' in r[ki]]
    s0 = starts[-1] if starts else 0
    ends = [i for i, r in enumerate(data) if i > s0 and 'k_fill<' in r[ki]]
    part = data[s0:(ends[0] + 1 if ends else len(data))]
    print(f"# last solve: launches {s0}..{s0 + len(part) - 1} of {len(data)}")
else:
    part = data
agg = collections.OrderedDict()
for r in part:
    name = r[ki].split('(')[0][:56]
    a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += float(r[vi].replace(',', ''))
tot = sum(v[1] for v in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:24]:
    print(f"{k:56s} {c:4d} {t/1e6:9.3f} ms {100*t/tot:5.1f}%")
print(f"total {tot/1e6:.3f} ms, {len(part)} launches")
