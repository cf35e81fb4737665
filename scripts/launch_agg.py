"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv, collections, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == 'ID':
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    n = re.sub(r'\(.*', '', d['Kernel Name'])[:60]
    agg[n][0] += 1
    agg[n][1] += float(d['Metric Value'].replace(',', '')) * scale.get(d['Metric Unit'], 1e-3)
tot = sum(t for _, t in agg.values())
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:50s} {c:6d} {t / 1e3:9.3f} ms {100 * t / tot:5.1f}%  avg {t / c:9.2f} us")
