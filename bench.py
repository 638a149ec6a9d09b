#!/usr/bin/env python
"""Decode throughput of the B200 PipeMax decode path (one JSON line).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (N=1): BASELINE.json configs[1] -- Qwen3-8B shape (36 layers,
d=4096, GQA 32/8, hd=128, ffn 12288, V=151936, random init, bf16), 256
requests, prompt 512 / gen 512, 2 cyclic micro-batches (~128 rows each),
block-first KV pool capped at 75% of the batch's peak KV so the scheduler
offloads/prefetches through pinned host memory.  On one GPU the pipeline is
PP=1 (every layer on the GPU); with N>1 under torchrun each rank runs an
independent replica of the same workload (replicas; the PP path is
``pipeline.py``).  A "step" is one rotation iteration of the reference engine
(REF pipeline_sim.py:386-543): plan + prefetch + one micro-batch through all
layers + offload.  Inputs > L2 (weights 16 GB, KV > 10 GB per step).

The reference arm (``--impl reference``) times the CPU implementation of the
path -- the fp32 numpy oracle port of the same decode step (the reference
itself has no model math) -- on all host threads, on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p, "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


# ---------------------------------------------------------------- workload
def workload(spec_name="qwen3-8b", n_req=256, prompt=512, gen=512, m=2, cap_frac=0.75, resident_frac=0.75):
    from paper_2605_02189_b200.workloads import decode_workload
    return decode_workload(spec_name, n_req, prompt, gen, m, cap_frac, resident_frac)


# BASELINE configs run as ONE pipeline stage on this GPU (--config):
# name, model, batch, prompt, gen, micro-batches, stage index
STAGE_CONFIGS = {
    "c3-stage": ("C3", "qwen3-32b", 512, 1024, 64, 8, 3),
    "c4-stage": ("C4", "llama3-70b", 256, 1024, 64, 8, 3),
}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock and throttle reasons sampled every 20 ms by NVML while the
    timed region runs (nvidia-smi one-shot queries as a fallback)."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu=0):
        self.samples, self.stop = [], threading.Event()
        self.gpu = gpu
        self.max_mhz = None

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self.stop.is_set():
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), int(get_r(h))))
                self.stop.wait(0.02)
            return
        except Exception:
            pass
        q = "clocks.sm,clocks.max.sm"
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip().split(",")
                self.max_mhz = float(out[1])
                self.samples.append((float(out[0]), 0))
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        time.sleep(0.1)
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        sm = sorted(x[0] for x in self.samples)
        reasons = set()
        for _, r in self.samples:
            for bit, name in self.REASONS.items():
                if r & bit:
                    reasons.add(name)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- CPU leg
def cpu_port_step_seconds(spec, M, ctx, layers_sample=1, seed=0):
    """Time the fp32 numpy oracle port of one decode step on a bounded
    sample: ``layers_sample`` full decoder layers for M rows at context
    ``ctx`` (attention per request, unbatched KV), plus lm_head; scaled to the
    whole model.  Returns (seconds per step, threads, sample description)."""
    import numpy as np
    from oracle import forward_ref as ref
    rng = np.random.default_rng(seed)
    d, H, Hkv, hd, f = spec.d, spec.H, spec.Hkv, spec.hd, spec.ffn
    W = lambda *s: (rng.standard_normal(s, dtype=np.float32) * 0.02)
    wq, wk, wv, wo = W(H * hd, d), W(Hkv * hd, d), W(Hkv * hd, d), W(d, H * hd)
    wg, wu, wd = W(f, d), W(f, d), W(d, f)
    x = rng.standard_normal((M, d), dtype=np.float32)
    K = rng.standard_normal((ctx, Hkv, hd), dtype=np.float32)
    V = rng.standard_normal((ctx, Hkv, hd), dtype=np.float32)
    nw = np.ones(d, np.float32)
    t0 = time.perf_counter()
    for _ in range(layers_sample):
        h = ref.rmsnorm(x, nw, spec.eps)
        q = (h @ wq.T).reshape(M, H, hd)
        _ = h @ wk.T, h @ wv.T
        o = np.stack([ref.attend(q[r], K, V, H // Hkv) for r in range(M)])
        x = x + o.reshape(M, -1) @ wo.T
        h = ref.rmsnorm(x, nw, spec.eps)
        x = x + (ref.silu(h @ wg.T) * (h @ wu.T)) @ wd.T
    t_layer = (time.perf_counter() - t0) / layers_sample
    lm_rows = min(spec.vocab, 16384)
    lm = W(lm_rows, d)
    t1 = time.perf_counter()
    _ = x @ lm.T
    t_head = (time.perf_counter() - t1) * spec.vocab / lm_rows
    threads = int(os.environ.get("OMP_NUM_THREADS", 0)) or len(os.sched_getaffinity(0))
    sample = (f"{layers_sample} decoder layer(s) x {M} rows at context {ctx} + {lm_rows}/{spec.vocab} lm_head "
              f"rows, fp32 numpy oracle port, scaled x{spec.layers} layers")
    return t_layer * spec.layers + t_head, threads, sample


# ---------------------------------------------------------------- GPU leg
def run_ours(args):
    import numpy as np
    import torch
    from paper_2605_02189_b200 import ops
    from paper_2605_02189_b200.engine import DecodeEngine

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks, peaks_src = load_peaks()
    if world > 1:
        # PP = N: one rank per stage (NCCL P2P), micro-batches >= stages
        from paper_2605_02189_b200.pipeline import PipelineEngine
        spec, state, cfg, params, reqs, desc = workload(m=max(2, world))
        desc["parallelism"] = f"pp{world}"
        desc["workload"] = desc["workload"].replace("PP=1", f"PP={world}")
        peng = PipelineEngine(spec, state, cfg, params, reqs, rank=rank, world=world, device=f"cuda:{local}",
                              kv_init="random", timing=True, seed=0)
        eng = peng.eng
        eng.step = peng.step
    elif args.config in STAGE_CONFIGS:
        # one pipeline stage of a PP=8 BASELINE config on this GPU: the stage's
        # layers (a middle stage: no embedding / lm_head), its KV pool and host
        # replica, the 8-micro-batch rotation; one micro-batch at a time, as a
        # real stage runs them (no lanes).  tokens/s = the pipeline's steady-
        # state throughput if every stage ran at this stage's speed.
        name, spec_name, n_req, prompt, gen, m, stage = STAGE_CONFIGS[args.config]
        spec, state, cfg, params, reqs, desc = workload(spec_name, n_req, prompt, gen, m)
        desc["workload"] = (f"{name}: stage {stage} of PP=8 ({spec.layers // 8} of {spec.layers} layers of "
                            f"{spec_name}), {m} micro-batches x {n_req // m} rows, prompt {prompt}, KV pool capped "
                            f"at 75% of peak, 25% of requests start in host memory (offload on)")
        desc["parallelism"] = "pp8-stage"
        eng = DecodeEngine(spec, state, cfg, params, reqs, pp=8, local_stages=[stage], device=f"cuda:{local}",
                           kv_init="random", timing=True, seed=rank)
    else:
        spec, state, cfg, params, reqs, desc = workload()
        eng = DecodeEngine(spec, state, cfg, params, reqs, device=f"cuda:{local}", kv_init="random",
                           timing=True, seed=rank)
    ex, kv = eng.stages[0]
    # warmup
    for _ in range(args.warmup):
        assert eng.step() is not None
    torch.cuda.synchronize()
    ids_host = torch.zeros(2 * args.steps, eng.m_cap, dtype=torch.int32).pin_memory()
    # ---- (1) device-timed region: K pipelined steps through the engine (the
    # host control plane runs ahead of the GPU), CUDA events on the compute
    # stream, barrier + synchronize on both sides, max over ranks
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    tokens, h2d0, d2h0, rec0 = 0, kv.h2d_bytes, kv.d2h_bytes, len(kv.records)
    kv_tok_sum = 0
    start_ev, end_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        eng.begin_region(start_ev)
        for i in range(args.steps):
            work = eng.step()
            assert work is not None, "workload ended inside the timed region"
            tokens += len(work.rows)
            kv_tok_sum += sum(work.positions) + len(work.rows)
        eng.end_region(end_ev)
        torch.cuda.synchronize()
    dev_s = start_ev.elapsed_time(end_ev) * 1e-3
    h2d_b, d2h_b = kv.h2d_bytes - h2d0, kv.d2h_bytes - d2h0
    recs = kv.records[rec0:]
    # ---- (2) end-to-end region: the same public call a serving loop makes,
    # each step's greedy ids read back to pinned host memory and waited for
    # before the next step starts (host<->device copies inside the region)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_tok, meta_b, e2e_h2d0, e2e_d2h0 = 0, 0, kv.h2d_bytes, kv.d2h_bytes
    w0 = time.perf_counter()
    pending = None   # (event, ...) of the previous step's ids readback
    for i in range(args.steps):
        t = eng.t
        work = eng.step()
        assert work is not None, "workload ended inside the e2e region"
        M = len(work.rows)
        e2e_tok += M
        meta_b += (eng.bucket(M) * (eng.max_blocks + 3) + 2 + 2 * M * eng.stages[0][0].aws.max_chunks) * 4
        # the step's greedy ids -> pinned host memory on its own stream; the
        # host waits for step t-1's ids while step t runs (one micro-batch of
        # slack, as a serving loop with two micro-batches in flight does)
        lane_stream = eng.stages[-1][1].streams[eng.lane_of(t)]
        with torch.cuda.stream(lane_stream):
            ids_host[i, :M].copy_(eng.last_executor(t).out_ids[:M], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(lane_stream)
        if pending is not None:
            pending.synchronize()
        pending = ev
    if pending is not None:
        pending.synchronize()
    wall = time.perf_counter() - w0
    e2e_h2d, e2e_d2h = kv.h2d_bytes - e2e_h2d0, kv.d2h_bytes - e2e_d2h0
    if dist:
        t = torch.tensor([dev_s, wall], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s, wall = t.tolist()
    # offload hiding over the device-timed steps
    stall = h2d_busy = d2h_busy = 0.0
    for r in recs:
        if "ready" in r:
            stall += r["ready"].elapsed_time(r["start"]) * 1e-3
        if "h2d_start" in r:
            h2d_busy += r["h2d_start"].elapsed_time(r["h2d_end"]) * 1e-3
        if "d2h_start" in r:
            d2h_busy += r["d2h_start"].elapsed_time(r["d2h_end"]) * 1e-3
    busy = h2d_busy + d2h_busy
    hidden = 1.0 - stall / busy if busy > 0 else 1.0
    M_avg = tokens / args.steps
    launches = args.steps * (ex.kernels_per_step(eng.bucket(int(round(M_avg)))) + 1)  # + meta upload
    value = tokens / dev_s
    # decode roofline of the step: the slower of HBM bytes (weights
    # + the micro-batch's KV + new KV + activations) and evicted-KV bytes over
    # PCIe (measured H2D/D2H rates of this run)
    hbm_bytes = sum(e.step_bytes(int(round(M_avg)), int(kv_tok_sum / args.steps - M_avg)) for e, _ in eng.stages)
    t_hbm = hbm_bytes / (peaks["hbm_gbs"] * 1e9)
    bw_h2d = h2d_b / h2d_busy if h2d_busy > 0 else None
    bw_d2h = d2h_b / d2h_busy if d2h_busy > 0 else None
    t_pcie = max((h2d_b / args.steps) / bw_h2d if bw_h2d else 0.0, (d2h_b / args.steps) / bw_d2h if bw_d2h else 0.0)
    roof_tok_s = M_avg / max(t_hbm, t_pcie)
    out = {
        "metric": "offline decode tokens/sec (B200, KV offload on)",
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_s / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random-init weights seeded N(0,0.02), random KV, random first tokens)",
        "config": desc,
        "e2e": {"value": e2e_tok / wall, "unit": "tokens/s",
                "h2d_bytes_per_step": int((e2e_h2d + meta_b) / args.steps),
                "d2h_bytes_per_step": int((e2e_d2h + e2e_tok * 4) / args.steps),
                "note": "K further steps through the public engine API (DecodeEngine.step, the simulate_decode "
                        "loop), wall clock, each step's greedy ids copied to pinned host memory and waited for "
                        "by the host one step later (two micro-batches in flight); H2D = KV prefetch + step "
                        "metadata, D2H = KV offload + ids"},
        "kv_transfer_hidden_fraction": hidden,
        "kv_transfer": {"h2d_bytes": h2d_b, "d2h_bytes": d2h_b, "h2d_busy_s": h2d_busy,
                        "d2h_busy_s": d2h_busy, "exposed_stall_s": stall,
                        "h2d_GBps": bw_h2d / 1e9 if bw_h2d else None, "d2h_GBps": bw_d2h / 1e9 if bw_d2h else None},
        "decode_roofline": {"hbm_bytes_per_step": hbm_bytes, "t_hbm_ms": t_hbm * 1e3, "t_pcie_ms": t_pcie * 1e3,
                            "roofline_tok_s": roof_tok_s, "frac": value / roof_tok_s,
                            "peak_hbm_gbs": peaks["hbm_gbs"], "peak_source": peaks_src,
                            "note": "per step: weights once + the active micro-batch's KV + new KV + activations "
                                    "over HBM vs prefetch/offload bytes over PCIe at this run's measured rates"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }
    if args.kernel_timing:
        # instrumented pass: the next K steps launched eagerly with CUDA events
        # around every GEMM / attention launch on the compute stream
        timer = ops.KernelTimer()
        ops.TIMER = timer
        eng.serialize_lanes = True   # per-launch events must not see the other lane's kernels
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng.begin_region(a_ev)
        n_prof = 0
        for i in range(args.steps):
            if eng.step() is None:
                break
            n_prof += 1
        eng.end_region(b_ev)
        torch.cuda.synchronize()
        ops.TIMER = None
        eng.serialize_lanes = False
        prof_s = a_ev.elapsed_time(b_ev) * 1e-3
        summ = timer.summary()
        kinds = sorted(summ.items(), key=lambda kv_: -kv_[1]["seconds"])
        top, d = kinds[0]
        achieved = (d["bytes"] / d["launches"]) / (d["seconds"] / d["launches"]) / 1e9
        traffic = None   # DRAM bytes per launch of this kind from the committed ncu capture
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "traffic_latest.json")))
            traffic = tr.get(top, {}).get("dram_bytes_per_launch")
        except Exception:
            pass
        out["roofline"] = {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peaks["hbm_gbs"],
                           "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                           "algorithmic_bytes_per_launch": d["bytes"] / d["launches"],
                           "peak_source": peaks_src, "share_of_step": d["seconds"] / prof_s,
                           "per_kind": {k: {"launches": v["launches"], "GBps": v["bytes"] / v["seconds"] / 1e9,
                                            "us_per_launch": v["seconds"] / v["launches"] * 1e6,
                                            "share": v["seconds"] / prof_s} for k, v in summ.items()},
                           "note": f"CUDA events around each launch on the compute stream over {n_prof} further "
                                   "steps of the same run launched eagerly (the timed region replays CUDA "
                                   "graphs); achieved = algorithmic bytes per launch (GEMM: weights once + "
                                   "activations; attention: the micro-batch's KV once) / launch time; "
                                   "gemm = the stream-K kernel alone, gemm_fixup = its fused fixup/post kernel "
                                   "(an event recorded between the two launches)"}
    if rank == 0 and args.calibrate:
        # on-box fit of the planner's estimator (REF model_core.py:158-182) from
        # measured iterations of this engine; reported beside the analytic one
        # the bench plans with (timing engine: it overwrites sampled KV slots)
        from paper_2605_02189_b200.calibrate import calibrate_on_device, params_dict
        cp, samples, err = calibrate_on_device(eng, reps=3)
        out["estimator"] = {"planned_with": params_dict(params), "calibrated": params_dict(cp),
                            "max_rel_fit_err": err, "samples": len(samples)}
    if rank == 0 and not args.no_cpu_baseline:
        kv_ctx = int(np.mean([eng.control.state.lengths.get(r, 0) for r in range(len(reqs))]))
        M = int(round(tokens / args.steps))
        sec, thr, sample = cpu_port_step_seconds(spec, M, kv_ctx)
        out["cpu_baseline"] = {"value": M / sec, "unit": "tokens/s", "cores": thr, "kind": "port",
                               "sample": sample}
    if rank == 0:
        print(json.dumps(out))
    if dist:
        peng.finish()
        torch.cuda.synchronize()
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    """CPU implementation of the path (oracle port) on all host threads."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    spec, state, cfg, params, reqs, desc = workload()
    M = max(len(b) for b in state.batches)
    ctx = 512 + args.warmup
    times = []
    sample = None
    for _ in range(max(1, args.steps)):
        sec, thr, sample = cpu_port_step_seconds(spec, M, ctx)
        times.append(sec)
    sec = sum(times) / len(times)
    val = M / sec
    out = {"impl": "reference", "metric": "offline decode tokens/sec (B200, KV offload on)", "value": val,
           "unit": "tokens/s", "n_gpus": int(os.environ.get("WORLD_SIZE", 1)), "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": desc,
           "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": thr, "kind": "port", "sample": sample},
           "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=6)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-kernel-timing", dest="kernel_timing", action="store_false")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-calibrate", dest="calibrate", action="store_false")
    ap.add_argument("--config", default="c2", choices=["c2"] + sorted(STAGE_CONFIGS),
                    help="c2 (default): BASELINE configs[1] on one GPU; c3-stage / c4-stage: one PP=8 stage")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference"
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
