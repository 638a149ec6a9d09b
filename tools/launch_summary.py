"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel
launches / total / share / avg over the last `n` launches (one or more
steps).  usage: python tools/launch_summary.py launches.csv [n_last]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
data = [(r[iK], float(r[iV].replace(",", ""))) for r in rows[1:] if r[iM] == "gpu__time_duration.sum"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(data)
data = data[-n:]
agg = collections.OrderedDict()
for k, t in data:
    name = k.split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    d = agg.setdefault(name, [0, 0.0])
    d[0] += 1
    d[1] += t
tot = sum(v[1] for v in agg.values())
print(f"| kernel | launches | total us | share | avg us |\n|---|---|---|---|---|")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k} | {c} | {t / 1e3:.1f} | {100 * t / tot:.1f}% | {t / c / 1e3:.1f} |")
print(f"| total | {sum(v[0] for v in agg.values())} | {tot / 1e3:.1f} | | |")
