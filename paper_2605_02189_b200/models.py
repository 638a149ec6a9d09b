"""Model shapes of the BASELINE configs and seeded random-init weights.

Only shapes matter for the decode hot path (the reference has no model math,
SURVEY.md 8c); semantics follow HF Llama / Qwen3 (RMSNorm, rotate-half RoPE,
GQA, SwiGLU; Qwen3 adds per-head q/k RMSNorm).  Weights are N(0, 0.02)
(norm weights 1 + N(0, 0.05) so indexing bugs show), generated from a seeded
torch generator on the target device and rounded to bf16.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class ModelSpec:
    name: str
    d: int            # hidden size
    layers: int
    H: int            # query heads
    Hkv: int          # kv heads
    hd: int           # head dim
    ffn: int          # intermediate size
    vocab: int
    qk_norm: bool     # Qwen3 per-head q/k RMSNorm
    rope_theta: float
    eps: float
    lm_head_std: float = 0.02

    @property
    def qkv_out(self) -> int:
        return (self.H + 2 * self.Hkv) * self.hd

    def kv_bytes_per_token(self, layers=None) -> int:
        """bf16 K+V bytes of one token over ``layers`` (default: all)."""
        return (self.layers if layers is None else layers) * 2 * self.Hkv * self.hd * 2

    def layer_weight_bytes(self) -> int:
        d, q, o, f = self.d, self.qkv_out, self.H * self.hd, self.ffn
        return 2 * (q * d + d * o + 2 * f * d + d * f) + 2 * 2 * d + (2 * 2 * self.hd if self.qk_norm else 0)

    def weight_bytes(self) -> int:
        return self.layers * self.layer_weight_bytes() + 2 * 2 * self.vocab * self.d + 2 * self.d

    def with_layers(self, n: int) -> "ModelSpec":
        return ModelSpec(self.name + f"-L{n}", self.d, n, self.H, self.Hkv, self.hd, self.ffn,
                         self.vocab, self.qk_norm, self.rope_theta, self.eps, self.lm_head_std)


# tiny: builder's choice recorded in DESIGN.md (H=4, Hkv=2, hd=64, ffn=768, V=4096)
TINY = ModelSpec("tiny-llama", 256, 4, 4, 2, 64, 768, 4096, False, 10000.0, 1e-5)
QWEN3_8B = ModelSpec("qwen3-8b", 4096, 36, 32, 8, 128, 12288, 151936, True, 1e6, 1e-6)
QWEN3_32B = ModelSpec("qwen3-32b", 5120, 64, 64, 8, 128, 25600, 151936, True, 1e6, 1e-6)
LLAMA3_70B = ModelSpec("llama3-70b", 8192, 80, 64, 8, 128, 28672, 128256, False, 5e5, 1e-5)

SPECS = {s.name: s for s in (TINY, QWEN3_8B, QWEN3_32B, LLAMA3_70B)}


def rope_table(spec: ModelSpec, max_pos: int) -> np.ndarray:
    """[max_pos][hd] fp32: cos in [:hd/2], sin in [hd/2:] (rotate-half RoPE).

    Computed in float64 and rounded once, so the GPU kernels and the oracle
    rotate with bit-identical coefficients."""
    half = spec.hd // 2
    inv = 1.0 / (spec.rope_theta ** (np.arange(half, dtype=np.float64) * 2.0 / spec.hd))
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.concatenate([np.cos(ang), np.sin(ang)], axis=1).astype(np.float32)


def init_layer_weights(spec: ModelSpec, layer: int, device, seed: int = 0) -> dict:
    """Logical (HF-layout) bf16 weights of one decoder layer: row-major
    [out, in]."""
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1_000_003 + 7919 * (layer + 1))

    def normal(*shape, std=0.02):
        return (torch.randn(*shape, generator=g, device=device, dtype=torch.float32) * std).to(torch.bfloat16)

    def norm_w(n):
        return (1.0 + torch.randn(n, generator=g, device=device, dtype=torch.float32) * 0.05).to(torch.bfloat16)

    w = {
        "attn_norm": norm_w(spec.d),
        "wq": normal(spec.H * spec.hd, spec.d),
        "wk": normal(spec.Hkv * spec.hd, spec.d),
        "wv": normal(spec.Hkv * spec.hd, spec.d),
        "wo": normal(spec.d, spec.H * spec.hd),
        "mlp_norm": norm_w(spec.d),
        "w_gate": normal(spec.ffn, spec.d),
        "w_up": normal(spec.ffn, spec.d),
        "w_down": normal(spec.d, spec.ffn),
    }
    if spec.qk_norm:
        w["q_norm"] = norm_w(spec.hd)
        w["k_norm"] = norm_w(spec.hd)
    return w


def init_embed(spec: ModelSpec, device, seed: int = 0) -> torch.Tensor:
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1_000_003 + 17)
    return (torch.randn(spec.vocab, spec.d, generator=g, device=device) * 0.02).to(torch.bfloat16)


def init_head(spec: ModelSpec, device, seed: int = 0) -> dict:
    g = torch.Generator(device=device)
    g.manual_seed(seed * 1_000_003 + 31)
    return {
        "final_norm": (1.0 + torch.randn(spec.d, generator=g, device=device) * 0.05).to(torch.bfloat16),
        "lm_head": (torch.randn(spec.vocab, spec.d, generator=g, device=device) * spec.lm_head_std).to(torch.bfloat16),
    }


def stage_layers(spec: ModelSpec, pp: int, stage: int) -> range:
    """Even layer split; earlier stages take the remainder."""
    base, extra = divmod(spec.layers, pp)
    start = stage * base + min(stage, extra)
    return range(start, start + base + (1 if stage < extra else 0))
