"""Stall samples and instructions of a one-kernel ncu report grouped by how often
each SASS instruction executed (= which warp role / loop level ran it).
Usage: python scripts/ncu_groups.py report.ncu-rep [top=14]"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))[1:]
h, d = rows[0], rows[1:]
e = h.index("Instructions Executed")
i = h.index("Warp Stall Sampling (All Samples)")
reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
tot = sum(float(r[i] or 0) for r in d)
totx = sum(float(r[e] or 0) for r in d)
g = collections.defaultdict(lambda: [0, 0, 0, collections.Counter()])
for r in d:
    if not r[e] or float(r[e]) == 0:
        continue
    x = int(float(r[e]))
    B = g[x]
    B[0] += 1
    B[1] += x
    B[2] += float(r[i] or 0)
    for rs in reasons:
        B[3][rs] += float(r[h.index(rs)] or 0)
print(f"warp-instructions {totx:.3g}, stall samples {tot:.0f}")
for x, (n, sx, ss, rc) in sorted(g.items(), key=lambda kv: -kv[1][2])[:int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
    print(f"exec {x:>10d} sites {n:4d} instr {100 * sx / totx:5.1f}% stalls {100 * ss / tot:5.1f}%",
          {k[6:]: int(v) for k, v in rc.most_common(3)})
