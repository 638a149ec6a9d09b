"""Per-kind summary of ONE decode step from an ncu launch list
(gpu__time_duration + dram bytes per launch): the launches between the last
two step-starting kernels (meta_upload), serialized by ncu (cold cache).
usage: python tools/launch_step_summary.py launches.csv [out.md]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
iI, iK, iM, iV = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = collections.OrderedDict()
for r in rows[1:]:
    d = per.setdefault(r[iI], {"k": r[iK]})
    d[r[iM]] = float(r[iV].replace(",", ""))
L = list(per.values())
starts = [i for i, d in enumerate(L) if "meta_upload" in d["k"]]
step = L[starts[-2]:starts[-1]]
agg = collections.OrderedDict()
for d in step:
    k = d["k"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    a = agg.setdefault(k, [0, 0.0, 0.0])
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0)
    a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
out = ["| kernel | launches | us total | share | us/launch | DRAM MB/launch | GB/s |", "|---|---|---|---|---|---|---|"]
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    out.append(f"| `{k}` | {a[0]} | {a[1] / 1e3:.1f} | {a[1] / tot:.3f} | {a[1] / a[0] / 1e3:.2f} | "
               f"{a[2] / a[0] / 1e6:.1f} | {a[2] / a[1]:.0f} |")
out.append(f"| total (serialized) | {sum(a[0] for a in agg.values())} | {tot / 1e3:.1f} | 1.000 | | | |")
txt = "\n".join(out)
print(txt)
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(txt + "\n")
