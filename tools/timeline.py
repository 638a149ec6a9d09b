"""Concurrent kernel timeline of the bench workload (CUPTI records via
torch.profiler over graph replays, lanes NOT serialised): how much of the
step has a weight/KV-streaming kernel (GEMM or attention) resident, how
much only latency-bound kernels (fixups, norms, metadata), how much
nothing; per-kind inclusive durations.  A PDL-launched kernel's record
starts at launch (its prologue overlaps the predecessor), so "streaming
kernel resident" is an upper bound on streaming time; the latency-only and
idle buckets are lower bounds on lost HBM time.
usage: python tools/timeline.py [config] [steps] [out.json]"""
import collections
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile
    config = sys.argv[1] if len(sys.argv) > 1 else "c2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    eng, _, spec, reqs, params, desc = bench.build_engine(config, calibrate=False)
    for _ in range(8):
        eng.step()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            eng.step()
        torch.cuda.synchronize()
    recs = []
    for e in prof.events():
        if getattr(e, "device_type", None) is None or str(e.device_type).split(".")[-1] != "CUDA":
            continue
        if "emcpy" in e.name or "emset" in e.name:
            continue
        kind = bench.kernel_kind(e.name) or "other"
        recs.append((e.time_range.start, e.time_range.end, kind, e.name))
    recs.sort()
    t0, t1 = recs[0][0], max(r[1] for r in recs)
    span = t1 - t0
    ev = []
    for s, e, kind, _ in recs:
        ev.append((s, 1, kind))
        ev.append((e, -1, kind))
    ev.sort(key=lambda x: (x[0], x[1]))
    active = collections.Counter()
    cover = collections.Counter()
    prev = t0
    for t, d, kind in ev:
        dt = t - prev
        if dt > 0:
            stream_n = active["gemm"] + active["attention"]
            small = sum(v for k, v in active.items() if k not in ("gemm", "attention"))
            if stream_n >= 2:
                cover["2+ streaming kernels"] += dt
            elif stream_n == 1:
                cover["1 streaming kernel"] += dt
            elif small:
                cover["only latency-bound kernels"] += dt
            else:
                cover["idle"] += dt
        active[kind] += d
        prev = t
    per = collections.defaultdict(lambda: [0, 0.0])
    for s, e, kind, _ in recs:
        per[kind][0] += 1
        per[kind][1] += e - s
    out = {"config": config, "steps": steps, "span_us": span, "us_per_step": span / steps,
           "coverage_us_per_step": {k: v / steps for k, v in cover.items()},
           "coverage_frac": {k: v / span for k, v in cover.items()},
           "per_kind": {k: {"launches_per_step": v[0] / steps, "incl_us_per_launch": v[1] / v[0]}
                        for k, v in per.items()}}
    print(json.dumps(out, indent=1))
    if len(sys.argv) > 3:
        json.dump(out, open(sys.argv[3], "w"), indent=1)


if __name__ == "__main__":
    main()
