"""Generate tests/golden/hf_*.npz: logits of ``transformers`` 5.5.0's own
Qwen3ForCausalLM / LlamaForCausalLM (eager attention, fp32) on this repo's
seeded random-init weights -- the pin for the forward oracles
(oracle/forward_ref.py, oracle/forward_seq.py; tests/test_oracle_hf.py).

Run once in the build container (transformers is importable there; the GPU
box never runs this):  python tests/golden/make_hf_golden.py

Cases (HF_CASES): the tiny C1 model at full depth, and one layer of each
BASELINE shape at its real d / H / Hkv / hd / ffn / rope / eps with the
vocabulary cut to 2048 rows (the vocabulary size only scales the lm_head).
Weights: models.init_layer_weights / init_embed / init_head on the CPU
generator (bf16-rounded), upcast to fp32 for HF.  Tokens: seeded uniform ids.
"""
import dataclasses
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2605_02189_b200.models import LLAMA3_70B, QWEN3_32B, QWEN3_8B, TINY  # noqa: E402

# name -> (spec, tokens, seed)
HF_CASES = {
    "tiny": (TINY, 48, 5),
    "qwen3_8b_l1": (dataclasses.replace(QWEN3_8B, name="qwen3-8b-l1v2k", layers=1, vocab=2048), 24, 6),
    "qwen3_32b_l1": (dataclasses.replace(QWEN3_32B, name="qwen3-32b-l1v2k", layers=1, vocab=2048), 24, 7),
    "llama3_70b_l1": (dataclasses.replace(LLAMA3_70B, name="llama3-70b-l1v2k", layers=1, vocab=2048), 24, 8),
}


def case_weights(spec, seed):
    """The CPU-generated weights of a case (bf16 tensors, HF layout)."""
    from paper_2605_02189_b200.models import init_embed, init_head, init_layer_weights
    layers = [init_layer_weights(spec, li, "cpu", seed) for li in range(spec.layers)]
    head = init_head(spec, "cpu", seed)
    return layers, init_embed(spec, "cpu", seed), head["final_norm"], head["lm_head"]


def case_tokens(spec, n, seed):
    return np.random.default_rng(1000 + seed).integers(0, spec.vocab, n)


def hf_logits(spec, layers, embed, final_norm, lm_head, tokens):
    from transformers import LlamaConfig, LlamaForCausalLM, Qwen3Config, Qwen3ForCausalLM
    common = dict(vocab_size=spec.vocab, hidden_size=spec.d, intermediate_size=spec.ffn,
                  num_hidden_layers=spec.layers, num_attention_heads=spec.H, num_key_value_heads=spec.Hkv,
                  head_dim=spec.hd, rms_norm_eps=spec.eps, max_position_embeddings=4096,
                  rope_parameters={"rope_theta": spec.rope_theta, "rope_type": "default"},
                  tie_word_embeddings=False, attention_bias=False, hidden_act="silu",
                  attn_implementation="eager", torch_dtype=torch.float32)
    if spec.qk_norm:
        model = Qwen3ForCausalLM(Qwen3Config(**common))
    else:
        model = LlamaForCausalLM(LlamaConfig(mlp_bias=False, **common))
    sd = {"model.embed_tokens.weight": embed, "model.norm.weight": final_norm, "lm_head.weight": lm_head}
    for li, w in enumerate(layers):
        p = f"model.layers.{li}."
        sd.update({p + "input_layernorm.weight": w["attn_norm"], p + "post_attention_layernorm.weight": w["mlp_norm"],
                   p + "self_attn.q_proj.weight": w["wq"], p + "self_attn.k_proj.weight": w["wk"],
                   p + "self_attn.v_proj.weight": w["wv"], p + "self_attn.o_proj.weight": w["wo"],
                   p + "mlp.gate_proj.weight": w["w_gate"], p + "mlp.up_proj.weight": w["w_up"],
                   p + "mlp.down_proj.weight": w["w_down"]})
        if spec.qk_norm:
            sd[p + "self_attn.q_norm.weight"] = w["q_norm"]
            sd[p + "self_attn.k_norm.weight"] = w["k_norm"]
    sd = {k: v.float() for k, v in sd.items()}
    missing, unexpected = model.load_state_dict(sd, strict=False)
    missing = [m for m in missing if "rotary" not in m]
    assert not missing and not unexpected, (missing, unexpected)
    model.eval()
    with torch.no_grad():
        out = model(torch.as_tensor(tokens, dtype=torch.long)[None])
    return out.logits[0].float().numpy()


def main():
    import transformers
    out_dir = os.path.dirname(os.path.abspath(__file__))
    torch.manual_seed(0)
    for name, (spec, n, seed) in HF_CASES.items():
        layers, embed, fnorm, head = case_weights(spec, seed)
        toks = case_tokens(spec, n, seed)
        lg = hf_logits(spec, layers, embed, fnorm, head, toks)
        np.savez_compressed(os.path.join(out_dir, f"hf_{name}.npz"), tokens=toks, logits=lg.astype(np.float32),
                            transformers=transformers.__version__, spec=spec.name)
        print(name, lg.shape, float(np.abs(lg).max()))


if __name__ == "__main__":
    main()
