"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): time per kernel."""
import collections
import csv
import io
import sys

text = open(sys.argv[1]).read()
text = text[text.index('"ID"'):]
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
for r in csv.DictReader(io.StringIO(text)):
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    agg[name][0] += 1
    agg[name][1] += float(r["Metric Value"].replace(",", "")) * scale[r["Metric Unit"]]
tot = sum(t for _, t in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"{k[:64]:64s} {n:6d} {t:10.1f} ms {100 * t / tot:5.1f}%  {t / n:8.3f} ms/launch")
print(f"total {tot:.1f} ms")
