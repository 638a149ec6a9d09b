"""Per-stage decode forward: the layers one pipeline rank owns, their block-
first KV pool and the kernel sequence of one micro-batch step.

Replaces the reference's simulated ``dur = actual / n`` stage slot
(REF pipeline_sim.py:423-427, :452-484) with real sm_100a kernels.  Per layer:

  rmsnorm(resid) -> QKV GEMM -> (q/k norm) RoPE + KV append -> paged attention
  -> O GEMM (+resid, fused epilogue) -> rmsnorm -> gate/up GEMM (SiLU*up fused
  epilogue) -> down GEMM (+resid, fused epilogue)

The residual stream stays fp32 on the device; GEMM operands are bf16.  All
buffers are allocated once (``m_cap`` rows) so the step can be captured in a
CUDA graph and replayed with new metadata.
"""

from __future__ import annotations

import math

import torch

from . import _C, ops
from .models import ModelSpec, init_embed, init_head, init_layer_weights, rope_table


def interleave_gate_up(w_gate: torch.Tensor, w_up: torch.Tensor) -> torch.Tensor:
    """Rows 2i = gate_i, 2i+1 = up_i so one 128-row GEMM tile holds matching
    gate/up pairs and the SiLU*up epilogue is a lane-pair shuffle."""
    return torch.stack([w_gate, w_up], dim=1).reshape(-1, w_gate.shape[1]).contiguous()


# L2 prefetch of the next projection's first weight bytes, issued by each
# GEMM's producers once their own loads are out (covers the fixup tail);
# MB per projection, 0 = off.  Single-lane engines only (with two lanes the
# other lane keeps HBM busy and the extra traffic competes).
import os as _os
PF_MB = float(_os.environ.get("PM_PF_MB", "0"))
PF_QKV = _os.environ.get("PM_PF_QKV", "0") == "1"
PF_STRIPES = _os.environ.get("PM_PF_STRIPES", "1") == "1"   # stripes at every next-GEMM worker's start   # QKV also prefetches O (across attention)


class StageExecutor:
    split_norm = False   # O/down fixup + separate RMSNorm kernel (set by the engine for one lane)
    fused = False        # split-K fixups inside the GEMM kernels (enable_fused; single-lane engines)

    def __init__(self, spec: ModelSpec, layers: range, *, first: bool, last: bool, m_cap: int,
                 pool_blocks: int, max_blocks: int, n_slots: int, device, seed: int = 0,
                 max_pos: int = 4096, weights=None, keep_logical=False, gemm_sms: int = None,
                 rows_hint: int = None):
        self.spec, self.layers = spec, list(layers)
        self.first, self.last = first, last
        self.L_s = len(self.layers)
        self.m_cap, self.max_blocks, self.dev = m_cap, max_blocks, device
        self.gemm_sms = gemm_sms
        self.rows_hint = rows_hint   # rows of a typical step (sizes the attention launch choice)
        s = spec
        self.logical = [] if keep_logical else None
        self.W = []
        for li in self.layers:
            w = weights[li] if weights is not None else init_layer_weights(s, li, device, seed)
            if keep_logical:
                self.logical.append(w)
            qkv = torch.cat([w["wq"], w["wk"], w["wv"]], 0).contiguous()
            self.W.append(dict(
                attn_norm=w["attn_norm"], mlp_norm=w["mlp_norm"],
                q_norm=w.get("q_norm"), k_norm=w.get("k_norm"),
                qkv=ops.Linear(qkv), o=ops.Linear(w["wo"].contiguous()),
                gu=ops.Linear(interleave_gate_up(w["w_gate"], w["w_up"])),
                down=ops.Linear(w["w_down"].contiguous())))
            if not keep_logical:
                del w
        self.embed = init_embed(s, device, seed) if first else None
        head = init_head(s, device, seed) if last else None
        self.final_norm = head["final_norm"] if last else None
        self.lm_head = ops.Linear(head["lm_head"]) if last else None
        self.lm_head_logical = head["lm_head"] if (last and keep_logical) else None
        self.rope = torch.from_numpy(rope_table(s, max_pos)).to(device)

        b16, i32 = torch.bfloat16, torch.int32
        # KV pool (block-first, token-major inside a block) -- shared by every lane
        self.tok_elems = self.L_s * 2 * s.Hkv * s.hd
        self.tok_bytes = self.tok_elems * 2
        self.block_bytes = 16 * self.tok_bytes
        self.pool_blocks = pool_blocks
        self.pool = torch.zeros(pool_blocks * 16 * self.tok_elems, dtype=b16, device=device)
        self.pool_map = ops.pool_tmap(self.pool, self.L_s, s.Hkv, s.hd)
        # greedy-token table indexed by request slot -- shared by every lane
        self.tok_table = torch.zeros(n_slots, dtype=i32, device=device)
        _C.call("pm_prepare_gemm")
        _C.call("pm_prepare_gemm_cl")
        _C.call("pm_prepare_attention")
        self._alloc_lane()

    def _alloc_lane(self):
        """Per-lane state: activations, step metadata, workspaces, graphs.  A
        lane is one micro-batch in flight; clone_lane() gives a second one
        that shares the weights, the KV pool and the token table."""
        s, m_cap, device = self.spec, self.m_cap, self.dev
        f32, b16, i32 = torch.float32, torch.bfloat16, torch.int32
        self.resid = torch.zeros(m_cap, s.d, dtype=f32, device=device)
        self.xn = torch.zeros(m_cap, s.d, dtype=b16, device=device)
        self.qkv = torch.zeros(m_cap, s.qkv_out, dtype=b16, device=device)
        self.q = torch.zeros(m_cap, s.H, s.hd, dtype=b16, device=device)
        self.attn = torch.zeros(m_cap, s.H * s.hd, dtype=b16, device=device)
        self.act = torch.zeros(m_cap, s.ffn, dtype=b16, device=device)
        # folded RMSNorm (cluster GEMM path): per-(128-feature tile, row) sums
        # of squares of the residual, written by the O/down epilogues and read
        # by the next projection's epilogue
        self.ssq = torch.zeros(s.d // 128, m_cap, dtype=f32, device=device)
        # split-K partial scratch of the cluster GEMMs (per lane: lanes run concurrently)
        self.cl_part = torch.empty(ops.CL_CTAS_MAX * 128 * 128, dtype=f32, device=device)
        self.xn_maps = ops.activation_maps(self.xn)
        self.attn_maps = ops.activation_maps(self.attn)
        self.act_maps = ops.activation_maps(self.act)
        self.block_table = torch.zeros(m_cap, self.max_blocks, dtype=i32, device=device)
        self.positions = torch.zeros(m_cap, dtype=i32, device=device)
        self.seq_lens = torch.ones(m_cap, dtype=i32, device=device)
        self.slots = torch.zeros(m_cap, dtype=i32, device=device)
        self.meta_dev = [self.block_table, self.positions, self.seq_lens, self.slots]
        self.prefill_tokens = torch.zeros(m_cap, dtype=i32, device=device)
        self.out_ids = torch.zeros(m_cap, dtype=i32, device=device)
        self.logits = None
        self.graphs = {}
        lins = [x[k] for x in self.W for k in ("qkv", "o", "gu", "down")] + ([self.lm_head] if self.last else [])
        for lin in lins:   # before the workspace is sized from the plans
            lin.sms = self.gemm_sms
        # one fixup-counter slice per GEMM call site of a step (4 per layer + lm_head)
        self.gws = ops.GemmWorkspace(m_cap, ops.GemmWorkspace.floats_needed(lins, m_cap),
                                     max(l.n_units for l in lins), self.lm_head.n_units if self.last else 1, device,
                                     sites=4 * self.L_s + 1)
        self.aws = ops.AttnWorkspace(m_cap, s.Hkv, s.hd, self.max_blocks, device, rows_hint=self.rows_hint)

    def enable_fused(self):
        """Every projection finishes its split units (and its fused epilogue:
        residual + next RMSNorm, q/k norm + RoPE + KV append, SiLU, logits +
        argmax) inside its own GEMM kernel -- one launch per projection.  The
        kernel's fixup tasks wait on other CTAs of the same grid, so this is
        for engines with ONE stream of dependent kernels (lanes == 1)."""
        for w in self.W:
            for k in ("qkv", "o", "gu", "down"):
                w[k].enable_fused(self.dev)
        if self.last:
            self.lm_head.enable_fused(self.dev)
        self.fused = True

    def clone_lane(self) -> "StageExecutor":
        """A second executor over the same weights, KV pool and token table
        with its own activations/metadata/workspaces/graphs, so two
        micro-batches can be in flight on two streams."""
        import copy
        twin = copy.copy(self)
        twin._alloc_lane()
        if self.logits is not None:
            twin.enable_logits()
        return twin

    # ------------------------------------------------------------------ views
    def pool_view(self):
        s = self.spec
        return self.pool.view(self.pool_blocks, 16, self.L_s, 2, s.Hkv, s.hd)

    def enable_logits(self):
        if self.last and self.logits is None:
            self.logits = torch.zeros(self.m_cap, self.spec.vocab, dtype=torch.float32, device=self.dev)

    # ------------------------------------------------------------------ forward
    def forward(self, M: int, stream=None, kv_tokens: int = 0, prefill_tokens: bool = False, layer_hook=None):
        """One micro-batch step of M rows (metadata already on the device).

        Stage 0 embeds ``tok_table[slots]``; later stages expect ``resid`` to
        hold the activations received from the previous stage.  The last
        stage writes greedy ids to ``out_ids`` and ``tok_table[slots]``."""
        s = self.spec
        if M == 0:
            return
        if ops.CL_GEMM and M <= ops.CL_MAX_M:
            return self._forward_cl(M, stream, prefill_tokens, layer_hook)
        if self.first:
            if prefill_tokens:   # prompt chunk: row m embeds prefill_tokens[m]
                ops.embed(self.prefill_tokens, None, self.embed, self.resid, M, stream)
            else:
                ops.embed(self.tok_table, self.slots, self.embed, self.resid, M, stream)
        # the stage's first norm; every later norm is fused into the residual
        # projection that precedes it (pm_gemm_resid_rmsnorm)
        ops.rmsnorm(self.resid, self.W[0]["attn_norm"], self.xn, M, s.eps, stream)
        pfb = int(PF_MB * 2**20) if self.split_norm else 0

        def pf(lin):   # (packed weight, bytes) of the projection that streams next
            if not pfb or lin is None:
                return None
            span = lin.packed.numel() * 2 if PF_STRIPES else 0
            return (lin.packed, min(pfb, lin.weight_bytes), span)
        for li, w in enumerate(self.W):
            nxt_w = self.W[li + 1] if li + 1 < len(self.W) else None
            # QKV projection + q/k norm + RoPE + paged KV append (one fused epilogue)
            w["qkv"].qkv_rope(self.xn_maps, M, self.qkv, self.gws, self.q, self.pool, self.block_table,
                              self.positions, self.rope, w["q_norm"], w["k_norm"], s.H, s.Hkv, s.hd, li, self.L_s,
                              s.eps, stream, prefetch=pf(w["o"]) if PF_QKV else None, site=4 * li)
            if layer_hook is not None:   # layer li's K/V is in the pool (prefill offload)
                layer_hook(li)
            ops.paged_attention(self.pool_map, self.q, self.block_table, self.seq_lens, self.attn, self.aws,
                                M, s.H, s.Hkv, s.hd, li, self.L_s, stream, kv_tokens=kv_tokens,
                                decode=not prefill_tokens)
            # O projection + residual + post-attention RMSNorm
            w["o"].resid_rmsnorm(self.attn_maps, M, self.resid, self.gws, w["mlp_norm"], self.xn, s.eps, stream,
                                 split_norm=self.split_norm, prefetch=pf(w["gu"]), site=4 * li + 1)
            w["gu"](self.xn_maps, M, ops.EPI_SILU_MUL, self.act, s.ffn, self.gws, stream, prefetch=pf(w["down"]),
                    site=4 * li + 2)
            # down projection + residual + the next norm (next layer's, or the final one)
            nxt = self.W[li + 1]["attn_norm"] if li + 1 < len(self.W) else (self.final_norm if self.last else None)
            nxt_lin = nxt_w["qkv"] if nxt_w is not None else (self.lm_head if self.last else None)
            if nxt is not None:
                w["down"].resid_rmsnorm(self.act_maps, M, self.resid, self.gws, nxt, self.xn, s.eps, stream,
                                        split_norm=self.split_norm, prefetch=pf(nxt_lin), site=4 * li + 3)
            else:
                w["down"](self.act_maps, M, ops.EPI_RESID_ADD, self.resid, s.d, self.gws, stream, site=4 * li + 3)
        if self.last:
            self.lm_head(self.xn_maps, M, ops.EPI_LOGITS_ARGMAX, self.logits, s.vocab, self.gws, stream,
                         site=4 * self.L_s)
            ops.argmax_reduce(self.gws, self.lm_head.n_units, M, self.out_ids, self.tok_table, self.slots, stream)

    def _forward_cl(self, M: int, stream, prefill_tokens: bool, layer_hook):
        """forward() on the cluster split-K GEMMs: every projection finishes
        its split-K reduction and its epilogue inside its own kernel, and the
        RMSNorm before gate/up, the next QKV and the lm_head is folded into
        the producing O/down epilogue (xn = bf16(x * w) + sum-of-squares
        partials) and the consuming GEMM's per-token scale.  5 launches per
        layer: QKV(+q/k norm, RoPE, KV append), attention, O(+resid),
        gate/up(+SiLU), down(+resid)."""
        s = self.spec
        if self.first:
            if prefill_tokens:
                ops.embed(self.prefill_tokens, None, self.embed, self.resid, M, stream)
            else:
                ops.embed(self.tok_table, self.slots, self.embed, self.resid, M, stream)
        ops.rmsnorm(self.resid, self.W[0]["attn_norm"], self.xn, M, s.eps, stream)
        rs = None   # the first QKV reads a normalised xn
        for li, w in enumerate(self.W):
            w["qkv"].cl(self.xn_maps, M, ops.CL_EPI_QKV_ROPE, stream, m_cap=self.m_cap, part=self.cl_part, rs=rs, eps=s.eps,
                        rope=dict(q_out=self.q, pool=self.pool, block_table=self.block_table, positions=self.positions,
                                  rope=self.rope, qn_w=w["q_norm"], kn_w=w["k_norm"], H=s.H, Hkv=s.Hkv, hd=s.hd,
                                  layer=li, L_s=self.L_s))
            if layer_hook is not None:
                layer_hook(li)
            ops.paged_attention(self.pool_map, self.q, self.block_table, self.seq_lens, self.attn, self.aws,
                                M, s.H, s.Hkv, s.hd, li, self.L_s, stream)
            w["o"].cl(self.attn_maps, M, ops.CL_EPI_RESID, stream, m_cap=self.m_cap, part=self.cl_part, resid=self.resid, norm_w=w["mlp_norm"],
                      xn=self.xn, ssq_out=self.ssq)
            w["gu"].cl(self.xn_maps, M, ops.CL_EPI_SILU, stream, m_cap=self.m_cap, part=self.cl_part, out=self.act, ld_out=s.ffn, rs=(self.ssq, s.d),
                       eps=s.eps)
            nxt = self.W[li + 1]["attn_norm"] if li + 1 < len(self.W) else (self.final_norm if self.last else None)
            w["down"].cl(self.act_maps, M, ops.CL_EPI_RESID, stream, m_cap=self.m_cap, part=self.cl_part, resid=self.resid, norm_w=nxt,
                         xn=self.xn if nxt is not None else None, ssq_out=self.ssq if nxt is not None else None)
            rs = (self.ssq, s.d) if nxt is not None else None
        if self.last:
            self.lm_head.cl(self.xn_maps, M, ops.CL_EPI_LOGITS, stream, m_cap=self.m_cap, part=self.cl_part, out=self.logits, ld_out=s.vocab, rs=rs,
                            eps=s.eps, ws=self.gws)
            ops.argmax_reduce(self.gws, self.lm_head.n_units, M, self.out_ids, self.tok_table, self.slots, stream)

    def run(self, M: int, stream, graphs: bool = True, kv_tokens: int = 0):
        """forward(M) on ``stream``; with ``graphs`` the whole kernel sequence
        for this M is captured once into a CUDA graph and replayed (the step's
        metadata lives in fixed device buffers, so replays see new rows)."""
        if not graphs or ops.TIMER is not None:
            self.forward(M, stream, kv_tokens=kv_tokens)
            return
        g = self.graphs.get(M)
        if g is None:
            g = self.capture(M, stream)
        with torch.cuda.stream(stream):
            g.replay()

    def capture(self, M: int, stream):
        """Record forward(M) into a CUDA graph (capture launches nothing)."""
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            self.forward(M, stream)
        self.graphs[M] = g
        return g

    def kernels_per_step(self, M: int = None) -> int:
        """Kernels of one forward(M): embed, the first RMSNorm, per layer the
        fused QKV (GEMM + norm/RoPE/append kernel), attention, the fused O and
        down projections (GEMM + reduce/residual/RMSNorm kernel each) and the
        gate/up GEMM (1-2 launches); lm_head (1-2) + argmax."""
        M = M or self.m_cap
        if ops.CL_GEMM and M <= ops.CL_MAX_M:
            return (1 if self.first else 0) + 1 + 5 * self.L_s + (2 if self.last else 0)
        if self.fused and M <= 256:   # one launch per projection + attention
            n = (1 if self.first else 0) + 1 + 5 * self.L_s
            return n + (2 if self.last else 0)
        n = (1 if self.first else 0) + 1 + self.L_s * (2 + 1 + 2 + 2)
        if self.split_norm:   # O / down: GEMM + reduce + a separate RMSNorm when the plan splits units
            n += sum((w["o"].launches(M) > 1) + (w["down"].launches(M) > 1) for w in self.W)
        n += sum(w["gu"].launches(M) for w in self.W)
        if not self.last:
            n += self.W[-1]["down"].launches(M) - 2
        else:
            n += 1 + self.lm_head.launches(M)
        return n

    # ------------------------------------------------------------------ roofline
    def gemm_bytes(self, M: int) -> int:
        """Algorithmic bytes of one step's projection GEMMs (bench.py's kernel
        roofline): each weight once, the bf16 activations in, the outputs
        (bf16; fp32 residual read + write and the normalised bf16 copy for
        O/down; logits fp32 when kept)."""
        tot = 0
        for w in self.W:
            for key, out_b in (("qkv", 2), ("o", 0), ("gu", 1), ("down", 0)):
                lin = w[key]
                tot += lin.weight_bytes + M * lin.k * 2 + (M * lin.n_out * out_b if out_b else M * lin.n_out * 10)
        if self.last:
            tot += self.lm_head.weight_bytes + M * self.lm_head.k * 2 + (M * self.spec.vocab * 4 if self.logits is not None else 0)
        return tot

    def attn_bytes(self, kv_tokens: int, M: int = 0) -> int:
        """Algorithmic bytes of one step's attention launches: every row's KV
        (``kv_tokens`` = sum of sequence lengths) once per layer, q in, o out."""
        s = self.spec
        return self.L_s * (kv_tokens * 2 * s.Hkv * s.hd * 2 + 2 * M * s.H * s.hd * 2)

    def step_bytes(self, M: int, kv_tokens: int) -> int:
        """Algorithmic HBM bytes of one step: weights once, the micro-batch's
        KV once per layer, new KV written once, activations (stated, small)."""
        s = self.spec
        w = sum(x["qkv"].weight_bytes + x["o"].weight_bytes + x["gu"].weight_bytes + x["down"].weight_bytes
                for x in self.W)
        if self.last:
            w += self.lm_head.weight_bytes
        kv = (kv_tokens + M) * self.tok_bytes
        act = self.L_s * M * (4 * s.d * 4 + 2 * (s.qkv_out + 2 * s.H * s.hd + s.ffn)) * 1
        return w + kv + act
