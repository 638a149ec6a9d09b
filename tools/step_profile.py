"""Decompose bench.py's step time: full engine step (device events), host
time per step, and bare graph replay of the same bucket back to back."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2605_02189_b200.engine import DecodeEngine  # noqa: E402

spec, state, cfg, params, reqs, desc = bench.workload()
eng = DecodeEngine(spec, state, cfg, params, reqs, device="cuda:0", kv_init="random", timing=True)
ex, kv = eng.stages[0]
for _ in range(6):
    eng.step()
torch.cuda.synchronize()
K = int(sys.argv[1]) if len(sys.argv) > 1 else 40
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
host = []
a.record(kv.compute)
Ms = []
for _ in range(K):
    t0 = time.perf_counter()
    w = eng.step()
    host.append(time.perf_counter() - t0)
    Ms.append(len(w.rows))
b.record(kv.compute)
torch.cuda.synchronize()
full = a.elapsed_time(b) / K
recs = kv.records[-K:]
per = []
for r in recs:
    c = r["start"].elapsed_time(r["end"]) if "start" in r and "end" in r else -1
    st = r["ready"].elapsed_time(r["start"]) if "ready" in r else -1
    h = r["h2d_start"].elapsed_time(r["h2d_end"]) if "h2d_start" in r else 0
    per.append(f"{r['M']}:{c:.2f}/{st:.2f}/{r.get('h2d_bytes', 0) / 1e6:.0f}MB@{h:.2f}")
print("per step M:compute_ms/stall_ms/h2d: " + " ".join(per))
print(f"full step: {full:.3f} ms/step (device), host {1e3*sum(host)/K:.3f} ms/step, M={sum(Ms)/K:.1f}")
Mb = eng.bucket(max(Ms))
g = ex.graphs[Mb]
for rep in range(2):
    a.record(kv.compute)
    with torch.cuda.stream(kv.compute):
        for _ in range(K):
            g.replay()
    b.record(kv.compute)
    torch.cuda.synchronize()
    print(f"graph replay bucket {Mb}: {a.elapsed_time(b) / K:.3f} ms/step")
# host-side cost per component (monkeypatched timers, GPU work still async)
import collections
acc = collections.defaultdict(float)


def timed(obj, name, key):
    fn = getattr(obj, name)

    def w(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        acc[key] += time.perf_counter() - t0
        return r
    setattr(obj, name, w)


timed(eng.control, "step", "control")
timed(kv, "prefetch", "prefetch")
timed(kv, "offload", "offload")
timed(kv, "before_compute", "before_compute")
timed(eng, "_upload_meta", "upload_meta")
timed(eng.meta, "next", "meta_ring_wait")
timed(eng, "_forward_all", "forward_launch")
n = 0
t0 = time.perf_counter()
for _ in range(K):
    if eng.step() is None:
        break
    n += 1
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print(f"host breakdown over {n} steps ({1e3 * tot / max(n, 1):.3f} ms/step wall): " +
      ", ".join(f"{k} {1e3 * v / max(n, 1):.3f}" for k, v in acc.items()))
# host cost of the control plane alone
t0 = time.perf_counter()
n = 0
for _ in range(K):
    if eng.control.step() is None:
        break
    n += 1
print(f"control plane alone: {1e3 * (time.perf_counter() - t0) / max(n, 1):.3f} ms/step")
# two micro-batches in flight: two graphs of the same bucket replayed on two
# streams concurrently (timing only -- they share activation buffers)
g2 = torch.cuda.CUDAGraph()
s2 = torch.cuda.Stream(priority=torch.cuda.Stream.priority_range()[1])
with torch.cuda.graph(g2, stream=s2):
    ex.forward(Mb, s2)
torch.cuda.synchronize()
for rep in range(2):
    a.record(kv.compute)
    s2.wait_event(a)
    for _ in range(K):
        with torch.cuda.stream(kv.compute):
            g.replay()
        with torch.cuda.stream(s2):
            g2.replay()
    e2 = torch.cuda.Event(enable_timing=True)
    e2.record(s2)
    kv.compute.wait_event(e2)
    b.record(kv.compute)
    torch.cuda.synchronize()
    print(f"two streams, bucket {Mb}: {a.elapsed_time(b) / (2 * K):.3f} ms per micro-batch step")
