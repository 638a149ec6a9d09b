"""Markdown table of the C5 sweep lines (gpurun_out/c5/*.json)."""
import glob
import json
import os
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c5"
rows = []
for f in glob.glob(os.path.join(src, "*.json")):
    try:
        d = json.loads(open(f).read())
    except Exception:
        continue
    c = os.path.basename(f)[:-5]
    bs, m = int(c.split("-bs")[1].split("-m")[0]), int(c.split("-m")[1])
    r = d["decode_roofline"]
    rows.append((bs, m, d["rows_per_step"], d["ms_per_step"], d["value"], r["frac"], r["t_hbm_ms"], r["t_pcie_ms"],
                 d["kv_transfer_hidden_fraction"], d["kv_transfer"]["h2d_GBps"], d["clocks"]["sm_mhz"]))
rows.sort()
print("| bs | micro-batches | rows/step | ms/step | tok/s (pipeline) | decode-roofline frac | t_hbm ms | t_pcie ms "
      "| KV transfer hidden | H2D GB/s | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for bs, m, rps, ms, v, fr, th, tp, hid, h2d, mhz in rows:
    print(f"| {bs} | {m} | {rps:.1f} | {ms:.3f} | {v:,.0f} | {fr:.3f} | {th:.3f} | {tp:.3f} | {hid:.3f} | "
          f"{(h2d or 0):.1f} | {mhz} |")
