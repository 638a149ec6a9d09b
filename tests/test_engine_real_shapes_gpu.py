"""End-to-end parity of the B200 decode engine at REAL model shapes against
the fp32 oracle (oracle/forward_seq.py, pinned to transformers 5.5.0 by
tests/test_oracle_hf.py).

Per case (tests/real_shapes.py): Qwen3-8B / Qwen3-32B at 2 layers and
Llama-3-70B at 1 layer with their full d / heads / hd / ffn / vocabulary;
240 (208) requests with prompts of 200-700 tokens prefilled by the real
prefill path, 3 micro-batches of ~64 rows, a KV-pool cap that forces plan
evictions and prefetches from pinned host memory, two lanes (micro-batches
in flight), CUDA graphs -- the code paths the bench runs (BN=128 tiles of the
stream-K GEMM, multi-chunk attention merges, q/k norm at GQA 8, lm_head +
argmax over the full vocabulary).

Tolerance (stated form).  At real widths the fp32 logits are O(1) (std
0.02*sqrt(d) = 1.3-1.8) and bf16 STORAGE alone -- fp32 math, bf16 rounding
wherever the engine stores a bf16 tensor (norm outputs, q/k/v, cached K/V,
attention output, SwiGLU activation) -- moves them by up to 0.08-0.16
(measured: the ``storage_bf16`` twin of oracle/forward_seq.py on the same
inputs), so the north star's example bound of 2e-2 max-abs is below what any
bf16-storage implementation reaches here.  The budget B = max-abs(twin - fp32)
is measured per case on these exact inputs, and the engine must add no error
beyond it, teacher-forced on its own tokens:
  * logits max-abs(engine - fp32) <= 1.25 B and rms(engine - fp32) <= 1.25
    rms(twin - fp32);
  * top-1 agreement with fp32 >= the twin's agreement - 1 % (and >= 96 %);
    no flip wherever the fp32 top-2 margin exceeds 2B;
  * free-running greedy ids over a 17-token horizon (the prefill token + 16
    decode steps) vs the fp32 oracle's own greedy decode: identical up to the
    first position where the oracle's top-2 margin is <= 2B.
The replica of every resident request equals its HBM blocks byte for byte
after the run's evict/prefetch round trips (checked in test_engine_gpu)."""
import numpy as np
import pytest
import torch

from oracle.forward_seq import SeqModel
from paper_2605_02189_b200.engine import DecodeEngine
from paper_2605_02189_b200.models import rope_table
from real_shapes import CASES, build_case

pytestmark = pytest.mark.gpu
TOL_FACTOR = 1.25
HORIZON = 16


def _oracle(eng, storage_bf16=False):
    spec = eng.spec
    layers = [w for ex, _ in eng.stages for w in ex.logical]
    ex0, exl = eng.stages[0][0], eng.stages[-1][0]
    hp = dict(d=spec.d, H=spec.H, Hkv=spec.Hkv, hd=spec.hd, qk_norm=spec.qk_norm, eps=spec.eps)
    return SeqModel(hp, layers, ex0.embed, exl.final_norm, exl.lm_head_logical, rope_table(spec, eng.max_pos),
                    device=eng.dev, chunk_tokens=8192, storage_bf16=storage_bf16)


@pytest.mark.parametrize("name", list(CASES))
def test_engine_real_shapes(name):
    spec, st, cfg, params, reqs, prompts = build_case(name)
    eng = DecodeEngine(spec, st, cfg, params, reqs, kv_init="prefill", prompts=prompts, record_logits="device",
                       seed=CASES[name][4], graphs=True)
    assert eng.lanes == 2
    first_tok = eng.stages[0][0].tok_table.cpu().numpy().copy()
    eng.run()
    assert eng.control.finished and eng.metrics.completed_requests == len(reqs)
    assert eng.n_evicted > 0 and eng.n_prefetched > 0
    rows_per_step = [len(r) for _, r, _, _ in eng.logits_log]
    assert max(rows_per_step) >= 64
    # the engine's per-request decode logits (on the device) and emitted ids
    per = {r: {} for r in reqs}
    for (t, rows, pos, lg), (_, _, ids) in zip(eng.logits_log, eng.ids_log):
        for i, r in enumerate(rows):
            per[r][pos[i]] = (lg, i, int(ids[i]))
    rids = sorted(reqs)
    seqs, want, emitted = [], [], {}
    for r in rids:
        P, g = reqs[r].input_len, reqs[r].output_len
        assert sorted(per[r]) == list(range(P, P + g)), r
        e = [int(first_tok[eng.slot_of[r]])] + [per[r][p][2] for p in range(P, P + g)]
        emitted[r] = e
        seqs.append(list(prompts[r]) + e[:g])
        want.append(list(range(P, P + g)))
    orc = _oracle(eng)
    twin = _oracle(eng, storage_bf16=True)
    st = {k: dict(worst=0.0, sq=0.0, n=0, agree=0, rows=0) for k in ("gpu", "twin", "gpu_twin")}
    per_pos = []   # (rid, pos, fp32 top-2 margin, gpu same, twin same)
    G = 24
    for g0 in range(0, len(rids), G):
        ref = orc.teacher_forced(seqs[g0:g0 + G], want[g0:g0 + G], numpy=False)
        tw = twin.teacher_forced(seqs[g0:g0 + G], want[g0:g0 + G], numpy=False)
        for j, r in enumerate(rids[g0:g0 + G]):
            got = torch.stack([per[r][p][0][per[r][p][1]] for p in want[g0 + j]])
            w, t = ref[j], tw[j]
            for k, (x, y) in (("gpu", (got, w)), ("twin", (t, w)), ("gpu_twin", (got, t))):
                e = (x - y).abs()
                st[k]["worst"] = max(st[k]["worst"], float(e.max()))
                st[k]["sq"] += float((e.double() ** 2).sum())
                st[k]["n"] += e.numel()
                st[k]["agree"] += int((x.argmax(-1) == y.argmax(-1)).sum())
                st[k]["rows"] += e.shape[0]
            top2 = torch.topk(w, 2, dim=-1).values
            margin = (top2[:, 0] - top2[:, 1]).tolist()
            g_same = (got.argmax(-1) == w.argmax(-1)).tolist()
            t_same = (t.argmax(-1) == w.argmax(-1)).tolist()
            per_pos += [(r, want[g0 + j][k], margin[k], g_same[k], t_same[k]) for k in range(len(margin))]
    for v in st.values():
        v["rms"] = (v["sq"] / v["n"]) ** 0.5
        v["top1"] = v["agree"] / v["rows"]
    # the bf16-storage error budget of THESE inputs: how far an ideal bf16
    # implementation (fp32 math, bf16 rounding exactly where the engine stores
    # bf16) lands from the fp32 reference
    budget = st["twin"]["worst"]
    band = 2 * budget
    flips = [(r, p, round(m, 4)) for r, p, m, g, _ in per_pos if not g]
    wide_flips = [f for f in flips if f[2] > band]
    # free-running greedy horizon vs the oracle's own greedy decode
    o_ids, o_margin = orc.greedy([prompts[r] for r in rids], HORIZON)
    full, diverged = 0, []
    for j, r in enumerate(rids):
        e = np.asarray(emitted[r][:HORIZON + 1])
        d = np.nonzero(e != o_ids[j])[0]
        if len(d) == 0:
            full += 1
            continue
        d = int(d[0])
        diverged.append((r, d, float(o_margin[j, d])))
    print(f"{name}: steps={len(rows_per_step)} rows/step max={max(rows_per_step)} evicted={eng.n_evicted} "
          f"prefetched={eng.n_prefetched}; logits vs fp32: engine max-abs {st['gpu']['worst']:.4g} rms "
          f"{st['gpu']['rms']:.3g} top1 {st['gpu']['top1']:.4f} | bf16-storage twin max-abs {budget:.4g} rms "
          f"{st['twin']['rms']:.3g} top1 {st['twin']['top1']:.4f} | engine vs twin max-abs "
          f"{st['gpu_twin']['worst']:.4g}; flips={len(flips)} (beyond the 2x-budget band {band:.3g}: "
          f"{len(wide_flips)}) {flips[:6]}; greedy {HORIZON + 1}-token horizon identical for {full}/{len(rids)}; "
          f"diverged (rid, at, margin)={diverged[:6]}")
    assert st["gpu"]["worst"] <= TOL_FACTOR * budget
    assert st["gpu"]["rms"] <= TOL_FACTOR * st["twin"]["rms"]
    assert st["gpu"]["top1"] >= st["twin"]["top1"] - 0.01
    assert st["gpu"]["top1"] >= 0.96
    assert not wide_flips, wide_flips
    for r, d, mg in diverged:
        assert mg <= band, (r, d, mg)
