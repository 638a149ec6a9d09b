"""Trace, metrics and block-count accounting types of the decode driver.

Mirrors the reference's ``pipeline_sim`` support types (REF = reference
``pkg/src/pipemax/pipeline_sim.py``): ``EventTrace`` (:57-96),
``EpisodeMetrics`` (:156-216), ``GpuState`` (:121-153), ``NoiseSpec``
(:99-118) and the error classes (:45-54).  On B200 the trace timestamps come
from CUDA events instead of a simulated clock; the schema (version 1, JSONL
with a header line) is unchanged so the reference's report tooling reads it.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

SCHEMA_VERSION = 1

# compute-end sorts before transfer-end before everything else at equal time
_KIND_ORDER = {"stage_compute_end": 0, "transfer_end": 1}


class ConfigError(ValueError):
    """Unusable cluster description (REF :45-46)."""


class OutOfMemory(RuntimeError):
    """Block accounting overdrawn -- a committed plan was infeasible; always a
    bug (REF :49-50)."""


class CapacityError(ValueError):
    """A request cannot fit in host KV memory (REF :53-54)."""


@dataclass
class SimEvent:
    time: float
    kind: str
    payload: dict
    seq: int = 0


class EventTrace:
    """Append-only event log with a deterministic final order (REF :65-96)."""

    def __init__(self):
        self.events = []
        self._seq = 0

    def emit(self, time, kind, **payload):
        self.events.append(SimEvent(time, kind, payload, self._seq))
        self._seq += 1

    def finalize(self):
        self.events.sort(key=lambda e: (e.time, _KIND_ORDER.get(e.kind, 2),
                                        e.payload.get("stage", -1), e.seq))

    def kinds(self):
        counts = {}
        for ev in self.events:
            counts[ev.kind] = counts.get(ev.kind, 0) + 1
        return counts

    def select(self, kind):
        return [ev for ev in self.events if ev.kind == kind]

    def to_jsonl(self, path, timestamp=None):
        head = {"schema_version": SCHEMA_VERSION, "kind": "trace_header"}
        if timestamp is not None:
            head["generated_at"] = timestamp
        lines = [json.dumps(head)]
        lines += [json.dumps({"time": ev.time, "kind": ev.kind, "payload": ev.payload})
                  for ev in self.events]
        with open(path, "w") as fh:
            fh.write("\n".join(lines) + "\n")


@dataclass(frozen=True)
class NoiseSpec:
    """Multiplicative noise of the reference's simulated durations
    (REF :99-118).  Accepted for signature compatibility; the B200 driver
    measures real durations and never samples it."""

    family: str = "normal"
    sigma: float = 0.02
    clip_sigmas: float = 3.0

    def __post_init__(self):
        if self.family not in ("normal", "none"):
            raise ValueError(f"unknown noise family {self.family!r}")
        if self.sigma < 0 or self.clip_sigmas <= 0:
            raise ValueError("sigma must be >= 0 and clip_sigmas > 0")

    def factor(self, rng) -> float:
        if self.family == "none" or self.sigma == 0:
            return 1.0
        lim = self.clip_sigmas * self.sigma
        return 1.0 + min(max(rng.normal(0.0, self.sigma), -lim), lim)


@dataclass
class GpuState:
    """Per-request block COUNTS of one stage's KV pool (REF :121-153).

    The physical allocator (``kv.BlockAllocator``) keeps one of these in
    lock-step so its counts can be compared with the reference's directly.
    """

    stage_id: int
    total_blocks: int
    free_blocks: int
    resident_blocks: dict = field(default_factory=dict)

    def allocate(self, rid, blocks: int):
        if blocks > self.free_blocks:
            raise OutOfMemory(f"request {rid} needs {blocks} blocks, only {self.free_blocks} free")
        self.free_blocks -= blocks
        self.resident_blocks[rid] = self.resident_blocks.get(rid, 0) + blocks

    def grow(self, rid):
        if self.free_blocks < 1:
            raise OutOfMemory(f"no free block for token growth of request {rid}")
        self.free_blocks -= 1
        self.resident_blocks[rid] += 1

    def release(self, rid):
        self.free_blocks += self.resident_blocks.pop(rid, 0)

    @property
    def used_blocks(self) -> int:
        return self.total_blocks - self.free_blocks


@dataclass
class EpisodeMetrics:
    """Outcome of a decode run (REF :156-216), plus B200 measurements
    (``hbm_roofline_fraction``, ``kv_transfer_hidden_fraction``, copy bytes)
    that the reference cannot produce."""

    total_tokens_generated: int = 0
    wall_seconds: float = 0.0
    tokens_per_second: float = 0.0
    prefill_seconds: float = 0.0
    decode_seconds: float = 0.0
    stall_seconds: float = 0.0
    prefetched_token_fraction: list = field(default_factory=list)
    exec_time_series: list = field(default_factory=list)
    exec_predicted_series: list = field(default_factory=list)
    iterations: int = 0
    completed_requests: int = 0
    steady_iteration: int = None
    max_active_batch_tokens: int = 0
    max_resident_tokens: int = 0
    max_kv_capacity_fraction: float = 0.0
    exposed_offload_seconds: float = 0.0
    phase_switches: int = 0
    growth_relief_evictions: int = 0
    # B200-only
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    h2d_busy_seconds: float = 0.0
    d2h_busy_seconds: float = 0.0
    kv_transfer_hidden_fraction: float = 1.0

    def finalize(self):
        self.tokens_per_second = (self.total_tokens_generated / self.wall_seconds
                                  if self.wall_seconds > 0 else 0.0)
        busy = self.h2d_busy_seconds + self.d2h_busy_seconds
        if busy > 0:
            self.kv_transfer_hidden_fraction = max(0.0, 1.0 - self.stall_seconds / busy)
        return self

    def to_record(self, policy: str = "dynamic", seed: int = 0, timestamp=None) -> dict:
        fr = self.prefetched_token_fraction
        rec = {
            "schema_version": SCHEMA_VERSION,
            "policy": policy,
            "seed": seed,
            "total_tokens_generated": self.total_tokens_generated,
            "wall_seconds": self.wall_seconds,
            "tokens_per_second": self.tokens_per_second,
            "prefill_seconds": self.prefill_seconds,
            "decode_seconds": self.decode_seconds,
            "stall_seconds": self.stall_seconds,
            "iterations": self.iterations,
            "completed_requests": self.completed_requests,
            "steady_iteration": self.steady_iteration,
            "mean_prefetched_token_fraction": sum(fr) / len(fr) if fr else 0.0,
            "max_active_batch_tokens": self.max_active_batch_tokens,
            "max_resident_tokens": self.max_resident_tokens,
            "max_kv_capacity_fraction": self.max_kv_capacity_fraction,
            "exposed_offload_seconds": self.exposed_offload_seconds,
            "phase_switches": self.phase_switches,
            "growth_relief_evictions": self.growth_relief_evictions,
            "h2d_bytes": self.h2d_bytes,
            "d2h_bytes": self.d2h_bytes,
            "kv_transfer_hidden_fraction": self.kv_transfer_hidden_fraction,
        }
        if timestamp is not None:
            rec["generated_at"] = timestamp
        return rec
