"""Per-kernel-kind DRAM traffic of one decode step from an ncu metrics CSV
(dram__bytes_read.sum, dram__bytes_write.sum, gpu__time_duration.sum over
the launches of the last `n` kernels).  Kinds match bench.py's roofline
kinds: "gemm" = the stream-K GEMM kernel, "gemm_fixup" = its post kernel, "attention".
usage: python tools/traffic_summary.py ncu.csv n_last out.json"""
import collections
import csv
import json
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
iI, iK, iM, iV = h.index("ID"), h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = collections.OrderedDict()
for r in rows[1:]:
    d = per.setdefault(r[iI], {"k": r[iK]})
    d[r[iM]] = float(r[iV].replace(",", ""))
launches = list(per.values())[-int(sys.argv[2]):]


def kind(name):
    if "gemm_stream" in name:
        return "gemm"
    if "gemm_" in name:
        return "gemm_fixup"
    if "paged_attn" in name:
        return "attention"
    return "other"


agg = collections.defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "ns": 0.0})
for d in launches:
    a = agg[kind(d["k"])]
    a["launches"] += 1
    a["dram_bytes"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    a["ns"] += d.get("gpu__time_duration.sum", 0)
out = {k: {"launches": v["launches"], "dram_bytes_per_launch": v["dram_bytes"] / v["launches"],
           "us_per_launch": v["ns"] / v["launches"] / 1e3} for k, v in agg.items()}
# bench.py's "gemm" kind times the GEMM call including its post/reduce kernel
if "gemm" in out and "gemm_fixup" in agg:
    g, p = agg["gemm"], agg["gemm_fixup"]
    out["gemm_call"] = {"launches": g["launches"],
                        "dram_bytes_per_launch": (g["dram_bytes"] + p["dram_bytes"]) / g["launches"]}
json.dump(out, open(sys.argv[3], "w"), indent=1)
print(json.dumps(out, indent=1))
