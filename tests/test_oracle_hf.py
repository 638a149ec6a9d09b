"""Pin the forward oracles to ``transformers`` 5.5.0 (CPU).

The reference has no model math, so the logits oracle restates
HF Qwen3 / Llama.  tests/golden/make_hf_golden.py ran HF's own
Qwen3ForCausalLM / LlamaForCausalLM (eager, fp32) on this repo's seeded
weights and committed the logits; here both restatements -- the per-token
numpy ``forward_ref`` and the matrix-form torch ``forward_seq`` -- must
reproduce them on the same weights and tokens."""
import os
import sys

import numpy as np
import pytest
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from make_hf_golden import HF_CASES, case_tokens, case_weights  # noqa: E402

from oracle.forward_ref import RefModel  # noqa: E402
from oracle.forward_seq import SeqModel  # noqa: E402
from paper_2605_02189_b200.models import rope_table  # noqa: E402

TOL = 1e-4   # fp32 vs fp32: summation order only


def _load(name):
    spec, n, seed = HF_CASES[name]
    g = np.load(os.path.join(HERE, "golden", f"hf_{name}.npz"))
    assert str(g["transformers"]) == "5.5.0"
    toks = case_tokens(spec, n, seed)
    assert np.array_equal(toks, g["tokens"])
    layers, embed, fnorm, head = case_weights(spec, seed)
    hp = dict(d=spec.d, layers=spec.layers, H=spec.H, Hkv=spec.Hkv, hd=spec.hd, ffn=spec.ffn, vocab=spec.vocab,
              qk_norm=spec.qk_norm, eps=spec.eps)
    return spec, hp, toks, g["logits"], layers, embed, fnorm, head


@pytest.mark.parametrize("name", sorted(HF_CASES))
def test_forward_seq_matches_hf(name):
    spec, hp, toks, want, layers, embed, fnorm, head = _load(name)
    m = SeqModel(hp, layers, embed, fnorm, head, rope_table(spec, 64))
    got = m.teacher_forced([toks], [list(range(len(toks)))])[0]
    err = float(np.abs(got - want).max())
    assert err <= TOL, err
    assert np.array_equal(got.argmax(-1), want.argmax(-1))


@pytest.mark.parametrize("name", ["tiny", "qwen3_8b_l1"])
def test_forward_ref_matches_hf(name):
    spec, hp, toks, want, layers, embed, fnorm, head = _load(name)
    f = lambda t: t.float().numpy()
    ref = RefModel(hp, [{k: f(v) for k, v in w.items()} for w in layers], f(embed), f(fnorm), f(head),
                   rope_table(spec, 64))
    caches = ref.new_cache()
    got = np.stack([ref.token_step(int(t), p, caches) for p, t in enumerate(toks)])
    err = float(np.abs(got - want).max())
    assert err <= TOL, err


def test_forward_seq_greedy_matches_token_loop():
    """The incremental (KV-cache) path of forward_seq equals its own
    teacher-forced pass on the greedy sequence."""
    spec, hp, toks, want, layers, embed, fnorm, head = _load("tiny")
    m = SeqModel(hp, layers, embed, fnorm, head, rope_table(spec, 128), chunk_tokens=64)
    prompts = [toks[:20], toks[5:37]]
    ids, margin = m.greedy(prompts, 8)
    for j, p in enumerate(prompts):
        seq = list(p) + list(ids[j, :8])
        lg = m.teacher_forced([seq], [list(range(len(p) - 1, len(seq)))])[0]
        assert np.array_equal(lg.argmax(-1), ids[j]), j
        assert np.all(margin[j] >= 0)
