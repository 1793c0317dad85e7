"""Per-kernel SM-time of the last full frame in an ncu multi-metric launch list (tools/prof_sm.sh)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith('==')]
h = rows[0]
recs = collections.OrderedDict()
for r in rows[1:]:
    if len(r) != len(h):
        continue
    d = dict(zip(h, r))
    k = recs.setdefault(d['ID'], {'name': d['Kernel Name']})
    k[d['Metric Name']] = d['Metric Value'].replace(',', '')
launches = list(recs.values())
idx = [i for i, d in enumerate(launches) if 'k_composite' in d['name']]
fr = launches[idx[-2] + 1:idx[-1] + 1]
agg = collections.OrderedDict()
tot_t = tot_c = 0
for d in fr:
    n = d['name'].split('(')[0][-48:]
    t = float(d['gpu__time_duration.sum']) / 1000
    c = float(d['sm__cycles_active.sum']) / 1e3
    a = agg.setdefault(n, [0, 0.0, 0.0, d.get('launch__grid_size'), d.get('launch__occupancy_limit_shared_mem'),
                           d.get('launch__occupancy_limit_registers'), d.get('sm__warps_active.avg.pct_of_peak_sustained_active')])
    a[0] += 1; a[1] += t; a[2] += c
    tot_t += t; tot_c += c
print(f"{'kcyc':>8} {'%':>5} {'us':>7}  n  grid  occ(smem,reg) warps%  kernel")
for n, (k, t, c, g, os_, orr, w) in sorted(agg.items(), key=lambda x: -x[1][2]):
    print(f"{c:8.0f} {100*c/tot_c:5.1f} {t:7.1f} {k:2d} {g:>5} {os_:>4},{orr:>3} {float(w):6.1f}  {n}")
print(f"total SM-active kcycles {tot_c:.0f}  (= {tot_c/148/1.965e3*1e3:.1f} us of the whole GPU at 1965 MHz); serialised {tot_t:.1f} us; launches {len(fr)}")
