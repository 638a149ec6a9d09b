"""Decode-control scenarios shared by the golden generator (which builds the
REFERENCE's objects) and the parity tests (which build ours).

Plain data only -- no imports of either package.  Each scenario is a dict:

  n            micro-batch count the scheduler rotates (``ClusterConfig.n``)
  requests     [(id, input_len, output_len, generated)]
  batches      initial resident partition as lists of ids (None = use
               ``initial_partition`` over ``resident``)
  resident     ids resident at start (used when batches is None)
  cfg          ClusterConfig kwargs (scheduling view)
  params       (alpha, beta, delta)
  knobs        SchedulerState knobs
  mode, quota  policy of ``_plan_step``
  horizon      iterations to run
"""

import math
import random

BLOCK = 16


def _cap_cfg(n, cap_blocks, kv_bytes, h2d=55e9, d2h=55e9, block=BLOCK):
    # capacity_blocks = (n*M - 0) // (bs*T) == cap_blocks exactly
    mem = -(-cap_blocks * block * kv_bytes // n)
    return dict(n=n, mem_per_gpu=mem, model_bytes=0, kv_bytes_per_token=kv_bytes,
                h2d_bandwidth=h2d, d2h_bandwidth=d2h, cpu_kv_capacity=10**15,
                block_size=block)


def _uniform(count, prompt, gen, start=0):
    return [(start + i, prompt, gen, 0) for i in range(count)]


def _random_reqs(count, seed, lo_in, hi_in, lo_out, hi_out):
    rng = random.Random(seed)
    return [(i, rng.randint(lo_in, hi_in), rng.randint(lo_out, hi_out), 0) for i in range(count)]


def _b200_params(kv_bytes, weight_bytes, hbm=6.5459e12):
    # alpha ~ 0 (weight-bound linears), beta = KV bytes/token over HBM,
    # delta = weight stream time
    return (1e-7, kv_bytes / hbm, weight_bytes / hbm)


def scenarios():
    out = {}
    tiny_kv = 4 * 2 * 2 * 64 * 2  # 4 layers, K+V, Hkv=2, hd=64, bf16 = 2048 B
    # C1: tiny, 4 micro-batches x 8 resident, pooled tail, pressure cap (App. B.8)
    reqs = _uniform(128, 128, 128)
    out["c1_tiny_pressure"] = dict(
        n=4, requests=reqs, batches=None, resident=list(range(32)),
        cfg=_cap_cfg(4, 300, tiny_kv), params=(1e-6, 1e-9, 4e-5),
        knobs=dict(ema_alpha=0.3), mode="dynamic", quota=0, horizon=400)
    reqs = _random_reqs(96, 11, 32, 128, 8, 96)
    out["c1_tiny_ragged"] = dict(
        n=4, requests=reqs, batches=None, resident=list(range(32)),
        cfg=_cap_cfg(4, 260, tiny_kv), params=(1e-6, 1e-9, 4e-5),
        knobs=dict(ema_alpha=None), mode="dynamic", quota=0, horizon=600)
    # C2: Qwen3-8B shape, 2 micro-batches, 256 x (512 + 512), capped pool
    q8_kv = 36 * 2 * 8 * 128 * 2
    reqs = _uniform(256, 512, 512)
    out["c2_qwen3_8b"] = dict(
        n=2, requests=reqs, batches=None, resident=list(range(192)),
        cfg=_cap_cfg(2, 192 * 40, q8_kv), params=_b200_params(q8_kv, 16.4e9),
        knobs=dict(ema_alpha=0.3), mode="dynamic", quota=0, horizon=300)
    # C3: Qwen3-32B shape, 8 micro-batches, 512 x 1024, inactive micro-batches offloaded
    q32_kv = 64 * 2 * 8 * 128 * 2
    reqs = _uniform(512, 1024, 64)
    out["c3_qwen3_32b"] = dict(
        n=8, requests=reqs, batches=None, resident=list(range(384)),
        cfg=_cap_cfg(8, 384 * 66, q32_kv), params=_b200_params(q32_kv, 65.5e9),
        knobs=dict(ema_alpha=0.3), mode="dynamic", quota=0, horizon=320)
    # C4: Llama-3-70B shape, 8 micro-batches, 256 x (1024 + 1024), KV beyond the cap
    l70_kv = 80 * 2 * 8 * 128 * 2
    reqs = _uniform(256, 1024, 1024)
    out["c4_llama70b"] = dict(
        n=8, requests=reqs, batches=None, resident=list(range(160)),
        cfg=_cap_cfg(8, 160 * 68, l70_kv), params=_b200_params(l70_kv, 141e9),
        knobs=dict(ema_alpha=0.3), mode="dynamic", quota=0, horizon=240)
    # C5: PP=4 Qwen3-32B sweep points (micro-batch count x batch size)
    for m, bs in ((4, 64), (8, 256), (16, 1024)):
        reqs = _random_reqs(bs, 100 + m, 256, 1024, 16, 128)
        res = list(range(bs * 3 // 4))
        cap = sum(-(-reqs[r][1] // BLOCK) + 2 for r in res)
        out[f"c5_m{m}_bs{bs}"] = dict(
            n=m, requests=reqs, batches=None, resident=res,
            cfg=_cap_cfg(m, cap, q32_kv), params=_b200_params(q32_kv, 65.5e9),
            knobs=dict(ema_alpha=0.3), mode="dynamic", quota=0, horizon=200)
    # eviction-heavy small states (n=3) and the two baseline policies
    reqs = _random_reqs(60, 21, 5, 60, 5, 40)
    for mode, quota in (("dynamic", 0), ("static", 120), ("none", 0)):
        out[f"small_n3_{mode}"] = dict(
            n=3, requests=reqs, batches=None, resident=list(range(12)),
            cfg=_cap_cfg(3, 70, 64, h2d=64 * 4000.0), params=(0.05, 0.01, 0.01),
            knobs=dict(ema_alpha=None, window_w=4), mode=mode, quota=quota, horizon=300)
    # single micro-batch (i == j == k) and bootstrap from an empty pipeline
    reqs = _random_reqs(20, 5, 10, 40, 4, 20)
    out["n1_single"] = dict(
        n=1, requests=reqs, batches=None, resident=list(range(6)),
        cfg=_cap_cfg(1, 40, 128, h2d=1e6), params=(1e-3, 1e-5, 1e-3),
        knobs=dict(), mode="dynamic", quota=0, horizon=200)
    out["bootstrap_empty"] = dict(
        n=4, requests=_random_reqs(30, 9, 40, 200, 4, 30), batches=None, resident=[],
        cfg=_cap_cfg(4, 120, 256, h2d=256 * 10.0), params=(1e-3, 1e-5, 1e-3),
        knobs=dict(ema_alpha=0.5), mode="dynamic", quota=0, horizon=300)
    return out


def set_digest(ids):
    """Short order-free digest of an id set (golden files stay small)."""
    import hashlib
    return hashlib.sha1(",".join(str(x) for x in sorted(ids)).encode()).hexdigest()[:16]
