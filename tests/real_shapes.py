"""Workloads of the real-shape engine parity tests (tests/test_engine_real_shapes_gpu.py),
kept import-light so the control-plane half is also checked on the CPU
(tests/test_real_shapes_plan.py): BASELINE model shapes at reduced depth,
>= 3 micro-batches of >= 64 rows, prompts 200-700 tokens (several attention
chunks per row), a KV-pool cap that forces plan evictions, growth relief and
prefetches from the pinned host pool."""
import dataclasses

import numpy as np

from paper_2605_02189_b200 import scheduler as sched
from paper_2605_02189_b200.model_core import ClusterConfig, EstimatorParams, Request, blocks_for_tokens
from paper_2605_02189_b200.models import LLAMA3_70B, QWEN3_32B, QWEN3_8B

# name -> (spec at reduced depth, requests, resident, micro-batches, seed)
CASES = {
    "qwen3_8b_l2": (QWEN3_8B.with_layers(2), 240, 192, 3, 11),
    "qwen3_32b_l2": (QWEN3_32B.with_layers(2), 240, 192, 3, 12),
    "llama3_70b_l1": (LLAMA3_70B.with_layers(1), 208, 192, 3, 13),
}
GEN = (17, 24)          # every request decodes >= 17 tokens: a 16-token free-running horizon after the first
PROMPT = (200, 700)


def build_case(name, slack=80):
    spec, n_req, n_res, m, seed = CASES[name]
    rng = np.random.default_rng(seed)
    reqs = {i: Request(i, int(rng.integers(*PROMPT)), int(rng.integers(*GEN))) for i in range(n_req)}
    prompts = {i: rng.integers(0, spec.vocab, reqs[i].input_len) for i in reqs}
    resident = list(range(n_res))
    batches = sched.initial_partition([reqs[r] for r in resident], m)
    st = sched.SchedulerState(n=m, batches=batches, lengths={r: q.prefix_len for r, q in reqs.items()},
                              gpu_resident=set(resident), cpu_pool=set(reqs) - set(resident),
                              ema_alpha=0.3, window_w=3, stability_threshold=0.5)
    kv = spec.kv_bytes_per_token()
    # the residents' prompt blocks plus ``slack``: tighter than their peak, so
    # growth forces evictions and the pooled requests wait for freed blocks
    cap = sum(blocks_for_tokens(reqs[r].input_len, 16) for r in resident) + slack
    cfg = ClusterConfig(n=m, mem_per_gpu=-(-cap * 16 * kv // m), model_bytes=0, kv_bytes_per_token=kv,
                        h2d_bandwidth=55e9, d2h_bandwidth=55e9, cpu_kv_capacity=10**15, block_size=16)
    # budget B*T/T_kv ~ a few requests per step
    params = EstimatorParams(1e-7, 1e-10, 3e-4 * kv / 8192)
    return spec, st, cfg, params, reqs, prompts
