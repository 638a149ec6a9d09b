"""Episode-level prefill <-> decode switching on the GPU (episode.B200Backend):
the B200 run makes exactly the decisions of the control-only run (which is
pinned to the reference by test_episode_golden.py) while really prefilling
with layer-wise offload, bulk-loading each decode phase's resident KV from
the host replicas and decoding; every request completes its tokens."""
import numpy as np
import pytest
import torch

from episode_scenarios import episode_scenarios

from paper_2605_02189_b200.episode import B200Backend, ControlBackend, run_episode
from paper_2605_02189_b200.model_core import ClusterConfig, EstimatorParams, Request
from paper_2605_02189_b200.models import TINY

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["ep_dynamic", "ep_n2_horizon"])
def test_episode_on_gpu_matches_control(name):
    sc = episode_scenarios()[name]
    cfg, params = ClusterConfig(**sc["cfg"]), EstimatorParams(*sc["params"])
    kw = dict(policy=sc["policy"], scheduler_knobs=dict(sc["knobs"]), rho_hi=sc["rho_hi"], horizon=sc["horizon"])
    wl_ref = [Request(rid, a, b, g) for rid, a, b, g in sc["requests"]]
    ctl = ControlBackend()
    m_ref = run_episode(wl_ref, cfg, params, backend=ctl, **kw)
    reqs = {rid: Request(rid, a, b, g) for rid, a, b, g in sc["requests"]}
    rng = np.random.default_rng(0)
    prompts = {r: rng.integers(0, TINY.vocab, q.input_len) for r, q in reqs.items()}
    gpu = B200Backend(TINY, cfg, params, reqs, prompts, seed=1)
    m = run_episode(list(reqs.values()), cfg, params, backend=gpu, **kw)
    assert gpu.phases == ctl.phases
    assert (m.iterations, m.total_tokens_generated, m.completed_requests, m.phase_switches) == \
        (m_ref.iterations, m_ref.total_tokens_generated, m_ref.completed_requests, m_ref.phase_switches)
    assert [reqs[r.id].generated for r in wl_ref] == [r.generated for r in wl_ref]
    assert gpu.tokens == m.total_tokens_generated
    assert m.prefill_seconds > 0 and m.decode_seconds > 0
    ids = gpu.eng.stages[0][0].tok_table[:len(reqs)].cpu()
    assert int(ids.min()) >= 0 and int(ids.max()) < TINY.vocab


def test_phase_start_loads_resident_kv_bit_exact():
    sc = episode_scenarios()["ep_dynamic"]
    cfg, params = ClusterConfig(**sc["cfg"]), EstimatorParams(*sc["params"])
    reqs = {rid: Request(rid, a, b, g) for rid, a, b, g in sc["requests"]}
    rng = np.random.default_rng(0)
    prompts = {r: rng.integers(0, TINY.vocab, q.input_len) for r, q in reqs.items()}
    gpu = B200Backend(TINY, cfg, params, reqs, prompts, seed=1)
    seen = []
    orig = gpu.eng.start_phase

    def check(control):
        orig(control)
        ex, kv = gpu.eng.stages[0]
        host = kv.rep.as_tensor()
        pool = ex.pool.view(torch.uint8).view(ex.pool_blocks, ex.block_bytes)
        for rid, blocks in control.alloc.tables.items():
            L = control.state.lengths[rid]
            off = kv.rep.offset(gpu.eng.slot_of[rid])
            dev = torch.cat([pool[b] for b in blocks]).cpu()[:L * ex.tok_bytes]
            assert torch.equal(dev, host[off:off + L * ex.tok_bytes]), rid
            seen.append(rid)
    gpu.eng.start_phase = check
    run_episode(list(reqs.values()), cfg, params, backend=gpu, policy="dynamic", horizon=60)
    assert seen
