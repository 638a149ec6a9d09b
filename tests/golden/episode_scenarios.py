"""Episode scenarios (prefill <-> decode switching) shared by the golden
generator (reference objects) and the parity test (ours).  Plain data only.

Host KV capacity (cpu_kv_capacity) is set small enough that the workload
needs several prefill/decode rounds; the GPU capacity (capacity_blocks) is
smaller still so decode phases start from remnants and prefetch."""

from scenarios import _cap_cfg, _random_reqs


def episode_scenarios():
    out = {}
    kv = 2048                                   # tiny model, bytes per token
    reqs = _random_reqs(40, 7, 20, 90, 8, 40)
    host_tokens = 1400                           # ~25 requests' prompts
    for name, policy in [("dynamic", "dynamic"), ("no_prefetch", "no_prefetch"), ("static", "static:0.5")]:
        cfg = _cap_cfg(4, 40, kv)
        cfg["cpu_kv_capacity"] = host_tokens * kv
        out[f"ep_{name}"] = dict(requests=reqs, cfg=cfg, params=(1e-6, 2e-8, 1e-4), policy=policy,
                                 rho_hi=0.9, horizon=None, knobs={})
    cfg = _cap_cfg(2, 24, kv)
    cfg["cpu_kv_capacity"] = 900 * kv
    out["ep_n2_horizon"] = dict(requests=_random_reqs(30, 11, 16, 60, 4, 30), cfg=cfg, params=(1e-6, 2e-8, 1e-4),
                                policy="dynamic", rho_hi=0.8, horizon=120, knobs={"window_w": 4})
    return out
