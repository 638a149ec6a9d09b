"""One-off probe of the GPU box: device props, host RAM, pinned H2D/D2H bandwidth."""
import os, time, json, subprocess
import torch
out = {}
out["nvidia_smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,memory.total,clocks.max.sm,pcie.link.gen.max,pcie.link.width.max", "--format=csv"], capture_output=True, text=True).stdout
out["meminfo"] = open("/proc/meminfo").read().splitlines()[:3]
out["cpus"] = len(os.sched_getaffinity(0))
out["cpu_model"] = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].strip()
p = torch.cuda.get_device_properties(0)
out["sms"] = p.multi_processor_count
out["mem_get_info"] = torch.cuda.mem_get_info()
res = {}
s = torch.cuda.Stream()
for sz in [16 << 10, 256 << 10, 1 << 20, 2 << 20, 8 << 20, 64 << 20, 256 << 20]:
    h = torch.empty(sz, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(sz, dtype=torch.uint8, device="cuda")
    reps = max(4, min(200, (1 << 30) // sz))
    for direction in ("h2d", "d2h"):
        with torch.cuda.stream(s):
            for _ in range(3):
                (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(reps):
                (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
            e1.record(s)
        s.synchronize()
        res[f"{direction}_{sz}"] = sz * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
out["pcie_GBps"] = res
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
