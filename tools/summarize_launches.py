"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr, data = rows[h], rows[h + 1:]
ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
scale = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in data:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].replace('void ', '').replace('bie::', '')
    tot[name] += float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':34s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:34s} {cnt[k]:8d} {v:10.3f} {v / T:7.3f}")
print(f"{'TOTAL':34s} {sum(cnt.values()):8d} {T:10.3f}")
