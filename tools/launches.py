"""Summarise an ncu launch list (gpu__time_duration.sum) for the last full frame."""
import collections, csv, sys
path = sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches.csv'
rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith('==')]
h = rows[0]
data = [dict(zip(h, r)) for r in rows[1:] if len(r) == len(h)]
idx = [i for i, d in enumerate(data) if 'k_composite' in d['Kernel Name']]
fr = data[idx[-2] + 1:idx[-1] + 1]
agg = collections.OrderedDict()
tot = 0
for d in fr:
    n = d['Kernel Name'].split('(')[0][-60:]
    t = float(d['Metric Value']) / 1000
    tot += t
    agg.setdefault(n, [0, 0.0])
    agg[n][0] += 1
    agg[n][1] += t
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{t:8.1f} us x{c:3d} {n}")
print('total', round(tot, 1), 'us; launches', len(fr))
