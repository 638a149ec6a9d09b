"""Synthetic decode workloads of the BASELINE configs: fixed
prompt/gen lengths, a KV-pool cap that forces offload, and the scheduling
view the reference engine expects (``initial_partition`` of the resident
requests, the rest in the host pool)."""

from __future__ import annotations

import math

from . import scheduler as sched
from .model_core import ClusterConfig, EstimatorParams, Request
from .models import SPECS

HBM_BYTES_PER_S = 6.5459e12   # planner's analytic B200 rate (calibrate.py fits the real one)


def decode_workload(spec_name="qwen3-8b", n_req=256, prompt=512, gen=512, m=2, cap_frac=0.75,
                    resident_frac=0.75):
    """(spec, SchedulerState, ClusterConfig, EstimatorParams, requests, description)."""
    spec = SPECS[spec_name]
    kv_tok = spec.kv_bytes_per_token()
    reqs = {i: Request(i, prompt, gen) for i in range(n_req)}
    peak_blocks = n_req * math.ceil((prompt + gen) / 16)
    cap = int(peak_blocks * cap_frac)
    # `resident_frac` of the batch starts in HBM; the rest waits in the pinned
    # host pool and is prefetched as the budget and free blocks allow
    resident = list(range(int(n_req * resident_frac)))
    batches = sched.initial_partition([reqs[r] for r in resident], m)
    state = sched.SchedulerState(n=m, batches=batches, lengths={r: q.prefix_len for r, q in reqs.items()},
                                 gpu_resident=set(resident), cpu_pool=set(reqs) - set(resident),
                                 ema_alpha=0.3)
    mem = -(-cap * 16 * kv_tok // m)
    cfg = ClusterConfig(n=m, mem_per_gpu=mem, model_bytes=0, kv_bytes_per_token=kv_tok,
                        h2d_bandwidth=55e9, d2h_bandwidth=55e9, cpu_kv_capacity=10**15, block_size=16)
    # B200 estimator: linears weight-bound (alpha~0), attention KV-bound
    params = EstimatorParams(1e-7, kv_tok / HBM_BYTES_PER_S, spec.weight_bytes() / HBM_BYTES_PER_S)
    desc = {"workload": f"{spec_name} decode, PP=1, {m} micro-batches, bs {n_req}, prompt {prompt} / gen {gen}, "
                        f"KV pool capped at {cap_frac:.0%} of peak, {1 - resident_frac:.0%} of requests start in "
                        f"host memory (offload on)",
            "model": spec_name, "global_batch": n_req, "seq_len": prompt + gen, "micro_batches": m,
            "pool_blocks": cap, "parallelism": "pp1", "l2": "inputs > L2 (weights + KV per step >> 126 MB)"}
    return spec, state, cfg, params, reqs, desc
