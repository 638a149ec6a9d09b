"""On-box calibration of the decode-time estimator.

The reference plans every step with ``estimate_decode_time(b, L) = alpha*b +
beta*L + delta`` (REF = reference ``pkg/src/pipemax``, model_core.py:148-155)
and fits (alpha, beta, delta) from profiled ``(b, L, seconds)`` samples with
``calibrate_estimator`` (model_core.py:158-182; ``pipemax-sim calibrate``,
cli.py:311-327).  Its prefetch budget ``B * T_hat`` (scheduler.py:84-93) is
only as good as that fit, so on B200 the samples come from the hardware:
``profile_samples`` times whole-pipeline decode iterations of the engine's own
stage executors (the CUDA graphs the decode loop replays) over a grid of batch
sizes and total prefix lengths, and ``calibrate_on_device`` fits them with the
same least-squares restatement.  ``write_samples_csv`` emits the reference's
CSV format, so the reference CLI can fit the same file.

Timing only: the sampled rows append KV at their synthetic positions inside
the engine's pool (run it on a timing engine or before seeding KV).
"""

from __future__ import annotations

import numpy as np
import torch

from .model_core import EstimatorParams, calibrate_estimator


def default_grid(m_cap: int, max_len: int):
    bs = sorted({b for b in (16, 32, 64, 128, 256) if b <= m_cap} | {m_cap})
    lens = sorted({x for x in (64, 256, 512, 1024) if x < max_len} | {max_len - 1})
    return [(b, b * per) for b in bs for per in lens]


def profile_samples(engine, grid=None, reps: int = 5, warmup: int = 2, seed: int = 0, pipelined: bool = None):
    """[(b, L, seconds)]: CUDA-event time of one decode iteration (every
    stage of ``engine``) with ``b`` rows whose prefix lengths sum to ``L``
    (equal per row), on synthetic block tables over the engine's pool.

    ``pipelined`` (default: the engine has several lanes): the STEP PERIOD of
    back-to-back iterations alternating over the lanes, as the decode loop
    runs them -- the time the planner's prefetch budget B * T_hat must cover
    (REF scheduler.py:84-93); otherwise one isolated iteration."""
    eng = engine
    lanes = eng.lanes if pipelined is None or pipelined else 1
    max_len = eng.max_blocks * 16 - 1
    grid = grid or default_grid(eng.m_cap, max_len)
    rng = np.random.default_rng(seed)
    n_blocks = eng.control.alloc.total
    kv0 = eng.stages[0][1]
    out = []
    for b, L in grid:
        per = max(1, min(max_len, L // b))
        nb = -(-(per + 1) // 16)
        tables = [list(rng.choice(n_blocks, nb, replace=nb > n_blocks)) for _ in range(b)]
        positions = [per] * b
        slots = [eng.trash_slot] * b
        for lane in range(lanes):
            eng._fill_meta(tables, positions, slots, lane=lane)
        torch.cuda.synchronize()
        times = []
        for i in range(warmup + reps):
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(kv0.streams[0])
            for st in kv0.streams[1:]:
                st.wait_event(a)
            n_it = 4 * lanes if lanes > 1 else 1
            for k in range(n_it):
                eng._forward_all(b, lane=k % lanes)
            for st in kv0.streams[1:]:
                ev = torch.cuda.Event()
                ev.record(st)
                kv0.streams[0].wait_event(ev)
            e.record(kv0.streams[0])
            torch.cuda.synchronize()
            if i >= warmup:
                times.append(a.elapsed_time(e) * 1e-3 / n_it)
        out.append((b, b * per, float(np.median(times))))
    return out


def calibrate_on_device(engine, grid=None, reps: int = 5, pipelined: bool = None):
    """Fit (alpha, beta, delta) to measured iterations; returns
    (EstimatorParams, samples, max relative fit error)."""
    samples = profile_samples(engine, grid, reps, pipelined=pipelined)
    params = calibrate_estimator(samples)
    err = max(abs(params.alpha * b + params.beta * L + params.delta - t) / t for b, L, t in samples)
    return params, samples, err


def step_errors(records):
    """(predicted, measured) step seconds of consecutive recorded steps: the
    planner's predicted step time vs the period end(t) - end(t-1)."""
    recs = sorted((r for r in records if "end" in r and r.get("info", {}).get("plan") is not None),
                  key=lambda r: r["t"])
    out = []
    for prev, cur in zip(recs, recs[1:]):
        if cur["t"] != prev["t"] + 1:
            continue
        meas = prev["end"].elapsed_time(cur["end"]) * 1e-3
        if meas > 0:
            out.append((cur["info"]["plan"].predicted_exec_seconds, meas))
    return out


def step_fidelity(records, t0: int = 0):
    """Per-step estimator fidelity of a decode run (the paper's claim, PAPER.md
    667-669): the planner's predicted step time vs the measured step period
    (end of step t minus end of step t-1, CUDA events on the compute streams)
    for every step after ``t0``.  Returns (fraction within 5 %, max relative
    error, steps compared)."""
    recs = sorted((r for r in records if "end" in r and r.get("info", {}).get("plan") is not None),
                  key=lambda r: r["t"])
    errs = []
    for prev, cur in zip(recs, recs[1:]):
        if cur["t"] != prev["t"] + 1 or cur["t"] < t0:
            continue
        meas = prev["end"].elapsed_time(cur["end"]) * 1e-3
        pred = cur["info"]["plan"].predicted_exec_seconds
        if meas > 0:
            errs.append(abs(pred - meas) / meas)
    if not errs:
        return None, None, 0
    errs = np.asarray(errs)
    return float((errs <= 0.05).mean()), float(errs.max()), len(errs)


def write_samples_csv(path: str, samples) -> None:
    """The reference's sample file: ``b,L,seconds`` rows (one header row)."""
    with open(path, "w") as fh:
        fh.write("b,L,seconds\n")
        for b, L, t in samples:
            fh.write(f"{int(b)},{int(L)},{t:.9e}\n")


def params_dict(p: EstimatorParams) -> dict:
    return {"alpha": p.alpha, "beta": p.beta, "delta": p.delta}
