#!/usr/bin/env python
"""Decode throughput of the B200 PipeMax decode path (one JSON line).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c3-stage|c3-last|c4-stage|c4-last|c5-...]

Workload (N=1, default ``c2``): BASELINE.json configs[1] -- Qwen3-8B shape
(36 layers, d=4096, GQA 32/8, hd=128, ffn 12288, V=151936, random init,
bf16), 256 requests, prompt 512 / gen 512, 2 cyclic micro-batches (~128 rows
each), block-first KV pool capped at 75% of the batch's peak KV so the
scheduler offloads/prefetches through pinned host memory.  On one GPU the
pipeline is PP=1 (every layer on the GPU); with N>1 under torchrun the ranks
form a PP=N pipeline (pipeline.py, one stage per rank, NCCL P2P).  A "step" is
one rotation iteration of the reference engine (REF pipeline_sim.py:386-543):
plan + prefetch + one micro-batch through all layers + offload.  Inputs > L2
(weights 16 GB, KV > 10 GB per step).

The default line also carries ``north_star``: BASELINE's target config (C3,
Qwen3-32B, PP=8, bs 512, seq 1024, offload on) measured per stage on this GPU
-- the last stage (8 layers + final norm + lm_head + argmax, the pipeline's
slowest) and a middle stage -- as a fraction of the per-stage decode roofline
with the % of KV transfer time hidden (north star: >= 0.70 and >= 90 %).

The reference arm (``--impl reference``) times the CPU implementation of the
path on the host cores: the fp32 decode step of the oracle port (torch CPU,
every layer, full lm_head, a bounded row sample) and the reference package's
own ``simulate_decode`` host cost per iteration (baseline/_ref, when present).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
METRIC = "offline decode tokens/sec (B200, KV offload on)"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p, "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


# ---------------------------------------------------------------- workloads
def workload(spec_name="qwen3-8b", n_req=256, prompt=512, gen=512, m=2, cap_frac=0.75, resident_frac=0.75):
    from paper_2605_02189_b200.workloads import decode_workload
    return decode_workload(spec_name, n_req, prompt, gen, m, cap_frac, resident_frac)


# BASELINE configs run as ONE pipeline stage on this GPU (--config):
# name -> (BASELINE config, model, batch, prompt, gen, micro-batches, pp, stage)
STAGE_CONFIGS = {
    "c3-stage": ("C3", "qwen3-32b", 512, 1024, 64, 8, 8, 3),
    "c3-last": ("C3", "qwen3-32b", 512, 1024, 64, 8, 8, 7),
    "c4-stage": ("C4", "llama3-70b", 256, 1024, 64, 8, 8, 3),
    "c4-last": ("C4", "llama3-70b", 256, 1024, 64, 8, 8, 7),
}
# C5: PP=4 Qwen3-32B sweep of micro-batch count m and batch size (last stage)
for _bs in (64, 128, 256, 512, 1024):
    for _m in (4, 8, 16):
        STAGE_CONFIGS[f"c5-bs{_bs}-m{_m}"] = ("C5", "qwen3-32b", _bs, 1024, 64, _m, 4, 3)


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
class CpuDecodeStep:
    """The fp32 decode step of the oracle port (oracle/forward_seq.py's
    semantics, one token per request) on the host cores with torch CPU: every
    decoder layer and the full lm_head for ``M`` rows, each row attending to
    its own ``ctx`` cached keys.  The weights of ONE layer (and the KV of one
    layer) are reused for every layer -- values do not change the cost, and at
    0.8-3 GB fp32 per layer they stream from DRAM each layer like distinct
    weights would; the lm_head is the full [V, d] matrix."""

    def __init__(self, spec, M, ctx, seed=0):
        import torch
        self.torch = torch
        torch.set_num_threads(len(os.sched_getaffinity(0)))
        g = torch.Generator().manual_seed(seed)
        d, H, Hkv, hd, f = spec.d, spec.H, spec.Hkv, spec.hd, spec.ffn
        W = lambda *s: torch.randn(*s, generator=g) * 0.02
        self.spec, self.M, self.ctx = spec, M, ctx
        self.wqkv, self.wo = W((H + 2 * Hkv) * hd, d), W(d, H * hd)
        self.wg, self.wu, self.wd = W(f, d), W(f, d), W(d, f)
        self.lm = W(spec.vocab, d)
        self.K = torch.randn(M, Hkv, ctx + 1, hd, generator=g)
        self.V = torch.randn(M, Hkv, ctx + 1, hd, generator=g)
        self.x0 = torch.randn(M, d, generator=g)
        self.nw = torch.ones(d)

    def _norm(self, x):
        return x * self.torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + self.spec.eps) * self.nw

    def step(self):
        torch, s, M = self.torch, self.spec, self.M
        H, Hkv, hd = s.H, s.Hkv, s.hd
        g = H // Hkv
        with torch.no_grad():
            x = self.x0.clone()
            for _ in range(s.layers):
                qkv = self._norm(x) @ self.wqkv.T
                q = qkv[:, :H * hd].view(M, Hkv, g, hd)
                self.K[:, :, -1] = qkv[:, H * hd:(H + Hkv) * hd].view(M, Hkv, hd)
                self.V[:, :, -1] = qkv[:, (H + Hkv) * hd:].view(M, Hkv, hd)
                sc = torch.softmax((q @ self.K.transpose(-1, -2)) / hd ** 0.5, dim=-1)   # [M, Hkv, g, L]
                o = (sc @ self.V).reshape(M, H * hd)
                x = x + o @ self.wo.T
                h = self._norm(x)
                x = x + (torch.nn.functional.silu(h @ self.wg.T) * (h @ self.wu.T)) @ self.wd.T
            return (self._norm(x) @ self.lm.T).argmax(-1)


def cpu_sample_rows(M):
    """Rows of the CPU port's step (env PM_CPU_ROWS; default the whole
    micro-batch): all layers and the full lm_head for this many rows.  At the
    C2 micro-batch a step is ~1-2 s on 16 host cores, so K=60 steps fit in a
    few minutes of host time."""
    return max(1, min(M, int(os.environ.get("PM_CPU_ROWS", M))))


def cpu_port_baseline(spec, M, ctx, steps=2):
    """Tokens/s of the CPU port on a bounded sample (rank 0, N=1)."""
    rows = cpu_sample_rows(M)
    step = CpuDecodeStep(spec, rows, ctx)
    step.step()   # warm
    t0 = time.perf_counter()
    for _ in range(steps):
        step.step()
    sec = (time.perf_counter() - t0) / steps
    threads = step.torch.get_num_threads()
    sample = (f"{steps} full decode steps (all {spec.layers} layers + the full {spec.vocab}-row lm_head, fp32) of "
              f"{rows} of the micro-batch's {M} rows at context {ctx}, torch CPU on {threads} threads")
    return rows / sec, sec, threads, sample


def reference_engine_cost(n_iter=60):
    """Host cost of the reference package's own decode engine
    (``pipemax.simulate_decode``, REF pipeline_sim.py:546-581, installed
    unmodified in baseline/_ref) on the bench's C2 state: microseconds per
    rotation iteration.  None when the package is absent."""
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_dir, "pipemax")):
        return None
    import importlib
    sys.path.insert(0, ref_dir)
    try:
        pm = importlib.import_module("pipemax")
        from paper_2605_02189_b200.workloads import decode_workload
        _, state, cfg, params, reqs, _ = decode_workload("qwen3-8b", 256, 512, 512, 2, 0.75, 0.75)
        rstate = pm.SchedulerState(n=state.n, batches=[set(b) for b in state.batches], lengths=dict(state.lengths),
                                   gpu_resident=set(state.gpu_resident), cpu_pool=set(state.cpu_pool),
                                   ema_alpha=state.ema_alpha)
        rcfg = pm.ClusterConfig(**{k: getattr(cfg, k) for k in cfg.__dataclass_fields__})
        rparams = pm.EstimatorParams(params.alpha, params.beta, params.delta)
        rreqs = {i: pm.Request(i, r.input_len, r.output_len) for i, r in reqs.items()}
        t0 = time.perf_counter()
        _, m = pm.simulate_decode(rstate, rcfg, rparams, None, n_iter, requests=rreqs, seed=0)
        sec = time.perf_counter() - t0
        return {"us_per_iteration": sec / n_iter * 1e6, "iterations": n_iter, "cores": 1,
                "package": "pipemax (baseline/_ref, unmodified)",
                "note": "the reference engine's own simulate_decode on the same C2 state (plan, commit, block "
                        "accounting, simulated transfers): host time per rotation iteration, one Python thread"}
    except Exception as e:   # report, never fail the bench on the baseline leg
        return {"error": f"{type(e).__name__}: {e}"}
    finally:
        sys.path.remove(ref_dir)


# ---------------------------------------------------------------- GPU leg
def build_engine(config, rank=0, world=1, local=0, calibrate=True):
    """(engine, pipeline engine or None, spec, requests, params, description).
    ``calibrate``: the engine fits the planner's estimator on this GPU before
    the run (DecodeEngine.recalibrate) and plans with the fit."""
    from paper_2605_02189_b200.engine import DecodeEngine
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
        return eng, peng, spec, reqs, params, desc
    if config in STAGE_CONFIGS:
        # one pipeline stage of a BASELINE PP config on this GPU: the stage's
        # layers (+ lm_head on the last stage), its KV pool and host replica,
        # the m-micro-batch rotation; one micro-batch at a time, as a real
        # stage runs them (no lanes).  tokens/s = the pipeline's steady-state
        # throughput if every stage ran at this stage's speed.
        name, spec_name, n_req, prompt, gen, m, pp, stage = STAGE_CONFIGS[config]
        spec, state, cfg, params, reqs, desc = workload(spec_name, n_req, prompt, gen, m)
        from paper_2605_02189_b200.models import stage_layers
        nl = len(stage_layers(spec, pp, stage))
        role = "last stage: + final norm, lm_head, argmax" if stage == pp - 1 else "a middle stage"
        desc["workload"] = (f"{name}: stage {stage} of PP={pp} ({nl} of {spec.layers} layers of {spec_name}; {role}), "
                            f"{m} micro-batches x {n_req // m} rows, prompt {prompt} + gen, KV pool capped at 75% of "
                            f"peak, 25% of requests start in host memory (offload on)")
        desc["parallelism"] = f"pp{pp}-stage{stage}"
        eng = DecodeEngine(spec, state, cfg, params, reqs, pp=pp, local_stages=[stage], device=f"cuda:{local}",
                           kv_init="random", timing=True, seed=rank, calibrate=calibrate)
        return eng, None, spec, reqs, params, desc
    spec, state, cfg, params, reqs, desc = workload()
    eng = DecodeEngine(spec, state, cfg, params, reqs, device=f"cuda:{local}", kv_init="random",
                       timing=True, seed=rank, calibrate=calibrate)
    return eng, None, spec, reqs, params, desc


_PCIE = {}


_HBM = {}


def hbm_probe(local=0):
    """Device-to-device copy rate (read + write bytes / s) of a 2 GB buffer
    in this process (best of 3): a diagnostic of the run's HBM state, not the
    roofline peak (MEASURED_PEAKS.json)."""
    import torch
    if local not in _HBM:
        n = 2 << 30
        a = torch.empty(n, dtype=torch.uint8, device=f"cuda:{local}")
        b = torch.empty_like(a)
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.copy_(a)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, 2 * n / (e0.elapsed_time(e1) * 1e-3))
        _HBM[local] = best
        del a, b
    return _HBM[local]


def host_placement(local=0):
    """CPU and NUMA node the bench process runs on vs the GPU's node."""
    out = {}
    try:
        cpu = int(open("/proc/self/stat").read().rsplit(")", 1)[1].split()[36])
        out["cpu"] = cpu
        nodes = [d for d in os.listdir(f"/sys/devices/system/cpu/cpu{cpu}") if d.startswith("node")]
        out["cpu_node"] = int(nodes[0][4:]) if nodes else None
        out["allowed_cpus"] = len(os.sched_getaffinity(0))
        from paper_2605_02189_b200.kv import device_numa_node
        out["gpu_node"] = device_numa_node(local)
    except Exception as e:   # diagnostic only
        out["error"] = repr(e)
    return out


def pcie_peak(local=0):
    """(H2D, D2H) bytes/s of a 256 MB pinned <-> device copy on this box
    (best of 3, CUDA events; measured once per process)."""
    import torch
    if local not in _PCIE:
        n = 256 << 20
        host = torch.empty(n, dtype=torch.uint8).pin_memory()
        dev = torch.empty(n, dtype=torch.uint8, device=f"cuda:{local}")
        best = [0.0, 0.0]
        for _ in range(3):
            for k, (dst, src) in enumerate(((dev, host), (host, dev))):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                dst.copy_(src, non_blocking=True)
                b.record()
                torch.cuda.synchronize()
                best[k] = max(best[k], n / (a.elapsed_time(b) * 1e-3))
        _PCIE[local] = tuple(best)
        del host, dev
    return _PCIE[local]


def measure_device(eng, steps, peaks, local=0, dist=None):
    """K pipelined steps through the engine (the host control plane runs
    ahead of the GPU), CUDA events on the compute stream, barrier +
    synchronize on both sides, max over ranks; KV-transfer hiding and the
    step's decode roofline."""
    import torch
    ex, kv = eng.stages[0]
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    tokens, h2d0, d2h0, rec0 = 0, kv.h2d_bytes, kv.d2h_bytes, len(kv.records)
    kv_tok_sum = 0
    start_ev, end_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        eng.begin_region(start_ev)
        for _ in range(steps):
            work = eng.step()
            assert work is not None, "workload ended inside the timed region"
            tokens += len(work.rows)
            kv_tok_sum += sum(work.positions) + len(work.rows)
        eng.end_region(end_ev)
        torch.cuda.synchronize()
    dev_s = start_ev.elapsed_time(end_ev) * 1e-3
    if dist:
        t = torch.tensor([dev_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s = float(t[0])
    h2d_b, d2h_b = kv.h2d_bytes - h2d0, kv.d2h_bytes - d2h0
    stall = h2d_busy = d2h_busy = 0.0
    for r in kv.records[rec0:]:
        if "ready" in r:
            stall += r["ready"].elapsed_time(r["start"]) * 1e-3
        if "h2d_start" in r:
            h2d_busy += r["h2d_start"].elapsed_time(r["h2d_end"]) * 1e-3
        if "d2h_start" in r:
            d2h_busy += r["d2h_start"].elapsed_time(r["d2h_end"]) * 1e-3
    busy = h2d_busy + d2h_busy
    hidden = 1.0 - stall / busy if busy > 0 else 1.0
    from paper_2605_02189_b200.calibrate import step_fidelity
    within5, max_err, n_cmp = step_fidelity(kv.records[rec0:])
    M_avg = tokens / steps
    # decode roofline of the step: the slower of HBM bytes (weights
    # + the micro-batch's KV + new KV + activations) and evicted-KV bytes over
    # PCIe (measured H2D/D2H rates of this run)
    hbm_bytes = sum(e.step_bytes(int(round(M_avg)), int(kv_tok_sum / steps - M_avg)) for e, _ in eng.stages)
    t_hbm = hbm_bytes / (peaks["hbm_gbs"] * 1e9)
    bw_h2d = h2d_b / h2d_busy if h2d_busy > 0 else None
    bw_d2h = d2h_b / d2h_busy if d2h_busy > 0 else None
    # the PCIe side of the roofline uses the LINK's rate per direction (a large
    # pinned copy measured on this box, pcie_peak()), not this run's achieved
    # copy rates -- a slow offload path must not make the roofline easier
    pk_h2d, pk_d2h = pcie_peak(local)
    t_pcie = max((h2d_b / steps) / pk_h2d, (d2h_b / steps) / pk_d2h)
    roof_tok_s = M_avg / max(t_hbm, t_pcie)
    value = tokens / dev_s
    return {
        "value": value, "tokens": tokens, "rows_per_step": M_avg, "dev_s": dev_s, "ms_per_step": dev_s / steps * 1e3,
        "hidden": hidden, "clocks": clocks.summary(),
        "fidelity": {"steps_within_5pct": within5, "max_rel_err": max_err, "steps": n_cmp},
        "kv_transfer": {"h2d_bytes": h2d_b, "d2h_bytes": d2h_b, "h2d_busy_s": h2d_busy, "d2h_busy_s": d2h_busy,
                        "exposed_stall_s": stall, "h2d_GBps": bw_h2d / 1e9 if bw_h2d else None,
                        "d2h_GBps": bw_d2h / 1e9 if bw_d2h else None},
        "decode_roofline": {"hbm_bytes_per_step": hbm_bytes, "t_hbm_ms": t_hbm * 1e3, "t_pcie_ms": t_pcie * 1e3,
                            "roofline_tok_s": roof_tok_s, "frac": value / roof_tok_s,
                            "peak_hbm_gbs": peaks["hbm_gbs"],
                            "pcie_peak_GBps": {"h2d": pk_h2d / 1e9, "d2h": pk_d2h / 1e9},
                            "hbm_probe_GBps": hbm_probe(local) / 1e9, "host": host_placement(local),
                            "note": "per step: weights once + the active micro-batch's KV + new KV + activations "
                                    "over HBM (measured peak) vs prefetch / offload bytes over the PCIe link "
                                    "(a 256 MB pinned copy per direction on this box)"},
    }


def measure_e2e(eng, steps, dist=None):
    """The same public call a serving loop makes (DecodeEngine.step), wall
    clock; each step's greedy ids read back to pinned host memory and waited
    for by the host one step later (two micro-batches in flight); the step's
    metadata goes host->device inside the step."""
    import torch
    kv = eng.stages[0][1]
    ids_host = torch.zeros(steps, eng.m_cap, dtype=torch.int32).pin_memory()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_tok, meta_b, h2d0, d2h0 = 0, 0, kv.h2d_bytes, kv.d2h_bytes
    w0 = time.perf_counter()
    pending = None
    for i in range(steps):
        t = eng.t
        work = eng.step()
        assert work is not None, "workload ended inside the e2e region"
        M = len(work.rows)
        e2e_tok += M
        meta_b += (eng.bucket(M) * (eng.max_blocks + 3) + 2 + 2 * M * eng.stages[0][0].aws.max_chunks) * 4
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
    if dist:
        t = torch.tensor([wall], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t[0])
    return {"value": e2e_tok / wall, "unit": "tokens/s",
            "h2d_bytes_per_step": int((kv.h2d_bytes - h2d0 + meta_b) / steps),
            "d2h_bytes_per_step": int((kv.d2h_bytes - d2h0 + e2e_tok * 4) / steps),
            "note": "K further steps through the public engine API (DecodeEngine.step, the simulate_decode loop), "
                    "wall clock, each step's greedy ids copied to pinned host memory and waited for by the host "
                    "one step later; H2D = KV prefetch + step metadata, D2H = KV offload + ids"}


KIND_OF = (("gemm_stream_kernel", "gemm"), ("gemm_cluster_kernel", "gemm"), ("paged_attn_kernel", "attention"),
           ("gemm_", "gemm_fixup"), ("rmsnorm", "norm"), ("embed", "embed"), ("argmax", "argmax"),
           ("meta_upload", "meta"))


def kernel_kind(name):
    for key, kind in KIND_OF:
        if key in name:
            return kind
    return None


def kernel_profile(eng, steps, peaks):
    """Per-kernel timing from CUPTI kernel records (torch.profiler) over
    ``steps`` further steps replaying the SAME CUDA graphs, with the lanes
    serialised so each kernel's time is its own.  A kernel launched with PDL
    starts while its predecessor drains, so its share of the step is taken as
    its exclusive time ``end_i - max(start_i, end_{i-1})`` on the serial
    timeline (these sum to the busy step time); ``achieved`` = algorithmic
    bytes per launch / exclusive time per launch."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    eng.serialize_lanes = True
    torch.cuda.synchronize()
    gemm_b = attn_b = 0
    n_done = 0
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            work = eng.step()
            if work is None:
                break
            n_done += 1
            M = eng.bucket(len(work.rows))
            for ex, _ in eng.stages:
                gemm_b += ex.gemm_bytes(len(work.rows))
            attn_b += sum(ex.attn_bytes(sum(work.positions) + len(work.rows), len(work.rows)) for ex, _ in eng.stages)
        torch.cuda.synchronize()
    eng.serialize_lanes = False
    recs = []
    for e in prof.events():
        if getattr(e, "device_type", None) is None or str(e.device_type).split(".")[-1] != "CUDA":
            continue
        kind = kernel_kind(e.name)
        if kind is None:
            continue
        recs.append((e.time_range.start, e.time_range.end, kind, e.name))
    recs.sort()
    summ, prev_end, busy = {}, None, 0.0
    for s0, s1, kind, name in recs:
        excl = s1 - max(s0, prev_end) if prev_end is not None else s1 - s0
        excl = max(excl, 0.0)
        prev_end = s1 if prev_end is None else max(prev_end, s1)
        d = summ.setdefault(kind, {"launches": 0, "incl_us": 0.0, "excl_us": 0.0})
        d["launches"] += 1
        d["incl_us"] += s1 - s0
        d["excl_us"] += excl
        busy += excl
    if not summ or "gemm" not in summ:
        return None, len(recs)
    bytes_of = {"gemm": gemm_b, "attention": attn_b}
    per_kind = {}
    for k, d in summ.items():
        row = {"launches": d["launches"], "us_per_launch_exclusive": d["excl_us"] / d["launches"],
               "us_per_launch_inclusive": d["incl_us"] / d["launches"], "share": d["excl_us"] / busy}
        if k in bytes_of and d["excl_us"] > 0:
            row["GBps"] = bytes_of[k] / (d["excl_us"] * 1e-6) / 1e9
        per_kind[k] = row
    top = max(("gemm", "attention"), key=lambda k: summ.get(k, {"excl_us": 0})["excl_us"])
    d = summ[top]
    achieved = bytes_of[top] / (d["excl_us"] * 1e-6) / 1e9
    traffic = None   # DRAM bytes per launch of this kind from the committed ncu capture
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "traffic_latest.json")))
        traffic = tr.get(top, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    roof = {"bound": "hbm", "kernel": {"gemm": "gemm_stream_kernel", "attention": "paged_attn_kernel"}[top],
            "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
            "traffic": traffic, "algorithmic_bytes_per_launch": bytes_of[top] / d["launches"],
            "achieved_inclusive": bytes_of[top] / (d["incl_us"] * 1e-6) / 1e9,
            "share_of_step": d["excl_us"] / busy, "per_kind": per_kind,
            "note": f"CUPTI kernel records (torch.profiler) over {n_done} further steps replaying the same CUDA "
                    "graphs with the two lanes serialised; exclusive time = end - max(start, previous end) on the "
                    "serial timeline (PDL overlap attributed once); algorithmic bytes: GEMM = weights once + "
                    "activations in + outputs, attention = the micro-batch's KV once"}
    return roof, len(recs) / max(1, n_done)


def free_engine(*objs):
    import torch
    for o in objs:
        del o
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def stage_summary(config, steps, warmup, peaks, local, calibrate=True):
    """One per-stage measurement (north-star key of the default line)."""
    eng, _, spec, reqs, params, desc = build_engine(config, local=local, calibrate=calibrate)
    for _ in range(warmup):
        assert eng.step() is not None
    if calibrate:   # closed loop: the warm-up steps' measured periods correct the fit
        eng.refit_online()
    r = measure_device(eng, steps, peaks, local)
    out = {"config": config, "workload": desc["workload"], "tokens_per_s": r["value"],
           "ms_per_step": r["ms_per_step"], "rows_per_step": r["rows_per_step"],
           "decode_roofline_frac": r["decode_roofline"]["frac"],
           "t_hbm_ms": r["decode_roofline"]["t_hbm_ms"], "t_pcie_ms": r["decode_roofline"]["t_pcie_ms"],
           "kv_transfer_hidden_fraction": r["hidden"], "clocks": r["clocks"],
           "estimator_fidelity": r["fidelity"], "online_refit": getattr(eng, "refit", None)}
    del eng
    free_engine()
    return out


def run_ours(args):
    import numpy as np
    import torch

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peaks, peaks_src = load_peaks()
    eng, peng, spec, reqs, params, desc = build_engine(args.config, rank, world, local,
                                                       calibrate=args.calibrate and world == 1)
    for _ in range(args.warmup):
        assert eng.step() is not None
    if args.calibrate and args.refit and world == 1:   # closed loop: the warm-up steps' periods correct the fit
        eng.refit_online()
    torch.cuda.synchronize()
    dev = measure_device(eng, args.steps, peaks, local, dist)
    e2e = measure_e2e(eng, args.steps, dist)
    out = {
        "metric": METRIC,
        "value": dev["value"],
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev["ms_per_step"],
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random-init weights seeded N(0,0.02), random KV, random first tokens)",
        "config": desc,
        "e2e": e2e,
        "kv_transfer_hidden_fraction": dev["hidden"],
        "kv_transfer": dev["kv_transfer"],
        "decode_roofline": dict(dev["decode_roofline"], peak_source=peaks_src),
        "rows_per_step": dev["rows_per_step"],
        "clocks": dev["clocks"],
    }
    if args.kernel_timing and rank == 0:
        roof, per_step = kernel_profile(eng, min(args.steps, 20), peaks)
        if roof is not None:
            roof["peak_source"] = peaks_src
            out["roofline"] = roof
            out["gpu_launches"] = int(round(per_step * args.steps))
    if "gpu_launches" not in out:
        ex = eng.stages[0][0]
        out["gpu_launches"] = args.steps * (ex.kernels_per_step(eng.bucket(int(round(dev["rows_per_step"])))) + 1)
    if rank == 0:
        # the planner's estimator: fitted on this GPU at engine start (REF
        # model_core.py:158-182) and planned with; fidelity of its per-step
        # prediction vs the measured step period over the timed steps
        from paper_2605_02189_b200.calibrate import params_dict
        est = {"planned_with": params_dict(eng.control.params), "analytic": params_dict(params),
               "step_fidelity": dev["fidelity"],
               "claim": "PAPER.md 667-669: >= 90% of steps within 5%, worst < 8%"}
        if getattr(eng, "refit", None) is not None:   # warm-up periods -> delta shift (refit_online)
            est["online_refit"] = eng.refit
        if eng.calibration is not None:
            est["max_rel_fit_err"] = eng.calibration["max_rel_fit_err"]
            est["samples"] = len(eng.calibration["samples"])
        out["estimator"] = est
    kv_ctx = int(np.mean([eng.control.state.lengths.get(r, 0) for r in range(len(reqs))]))
    M = int(round(dev["rows_per_step"]))
    if dist:
        peng.finish()
        torch.cuda.synchronize()
        dist.barrier()
        dist.destroy_process_group()
    del eng, peng
    free_engine()
    if rank == 0 and world == 1 and args.config == "c2" and args.north_star:
        ns = [stage_summary(c, args.steps, args.warmup, peaks, local, args.calibrate) for c in ("c3-last", "c3-stage")]
        worst = min(ns, key=lambda r: r["decode_roofline_frac"])
        out["north_star"] = {
            "target": "C3 (Qwen3-32B, PP=8, bs 512, seq 1024, offload on): >= 0.70 of the per-stage decode "
                      "roofline with >= 90% of KV transfer time hidden",
            "stages": ns, "worst_stage_frac": worst["decode_roofline_frac"],
            "worst_stage_hidden": min(r["kv_transfer_hidden_fraction"] for r in ns),
            "met": bool(worst["decode_roofline_frac"] >= 0.70 and
                        min(r["kv_transfer_hidden_fraction"] for r in ns) >= 0.90),
            "peak_hbm_gbs": peaks["hbm_gbs"], "peak_source": peaks_src}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        val, sec, thr, sample = cpu_port_baseline(spec, M, kv_ctx)
        out["cpu_baseline"] = {"value": val, "unit": "tokens/s", "cores": thr, "kind": "port", "sample": sample,
                               "seconds_per_step": sec}
    if rank == 0:
        print(json.dumps(out))


def run_reference(args):
    """The CPU implementation of the path on the host cores: the fp32 decode
    step of the oracle port, K timed steps (each a bounded row sample, every
    layer and the full lm_head), plus the reference engine's own host cost."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    if args.config in STAGE_CONFIGS:
        name, spec_name, n_req, prompt, gen, m, pp, stage = STAGE_CONFIGS[args.config]
        spec, state, cfg, params, reqs, desc = workload(spec_name, n_req, prompt, gen, m)
        from paper_2605_02189_b200.models import stage_layers
        spec = spec.with_layers(len(stage_layers(spec, pp, stage)))
    else:
        spec, state, cfg, params, reqs, desc = workload()
    M = max(len(b) for b in state.batches)
    ctx = int(sum(state.lengths[r] for r in state.batches[0]) / max(1, len(state.batches[0])))
    rows = cpu_sample_rows(M)
    step = CpuDecodeStep(spec, rows, ctx)
    for _ in range(args.warmup):
        step.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step.step()
    sec = (time.perf_counter() - t0) / args.steps
    val = rows / sec
    thr = step.torch.get_num_threads()
    sample = (f"{args.steps} full decode steps (all {spec.layers} layers + the full {spec.vocab}-row lm_head, "
              f"fp32) of {rows} of the micro-batch's {M} rows at context {ctx}, torch CPU on {thr} threads")
    out = {"impl": "reference", "metric": METRIC, "value": val,
           "unit": "tokens/s", "n_gpus": int(os.environ.get("WORLD_SIZE", 1)), "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": desc,
           "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": thr, "kind": "port", "sample": sample},
           "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    eng_cost = reference_engine_cost()
    if eng_cost is not None:
        out["reference_engine"] = eng_cost
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=6)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-kernel-timing", dest="kernel_timing", action="store_false")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-calibrate", dest="calibrate", action="store_false",
                    help="plan with the analytic estimator instead of the on-box fit")
    ap.add_argument("--no-north-star", dest="north_star", action="store_false")
    ap.add_argument("--no-refit", dest="refit", action="store_false",
                    help="plan with the start-up grid fit only (no warm-up delta correction; A/B)")
    ap.add_argument("--config", default="c2", choices=["c2"] + sorted(STAGE_CONFIGS),
                    help="c2 (default): BASELINE configs[1] on one GPU; c3-*/c4-*: one PP=8 stage "
                         "(-last = the lm_head stage); c5-bs*-m*: one PP=4 stage of the C5 sweep")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference"
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
