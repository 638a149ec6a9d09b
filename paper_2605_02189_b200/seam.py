"""The reference engine's injection seam, on B200 hardware.

The reference's decode loop ``_DecodeEngine`` (REF pkg/src/pipemax/
pipeline_sim.py:330-543) takes its block accounting and its two PCIe links
as duck-typed objects:

  gpu  : ``allocate(rid, blocks)``, ``grow(rid)``, ``release(rid)``,
         ``free_blocks``, ``total_blocks``, ``resident_blocks``
         (``GpuState``, pipeline_sim.py:121-153)
  h2d / d2h : ``submit_stream(when, total_bytes, chunk_bytes, tag) -> handle``,
         ``submit_high(when, n_bytes, tag) -> (start, end)``,
         ``finish_stream(handle) -> end``, ``drain()``, ``records``, ``name``,
         ``link.direction`` (``ChannelSim``, transfer.py:195-332)

``B200GpuState`` and ``B200CopyChannel`` implement them over a stage's real
block pool, host replica and CUDA copy streams, so the reference's own,
unmodified loop drives B200 KV traffic:

  * ``allocate``/``grow``/``release`` hand out PHYSICAL blocks of the pool
    (``control.BlockAllocator``) with the reference's count semantics
    (``OutOfMemory`` on overdraw);
  * a ``("kv_prefetch", rid, j)`` stream copies request ``rid``'s host-replica
    blocks into the physical blocks ``allocate`` just gave it (H2D, one DMA
    per run of consecutive blocks, on the channel's low-priority stream);
  * a ``("kv_offload_decode", t)`` stream moves the byte count the reference
    computes (the loop passes bytes, not rows) from a device staging area to
    pinned host memory;
  * ``submit_high`` (the activation hop) copies ``n_bytes`` on a
    high-priority stream;
  * times: the channel keeps the reference's FIFO link clock (``busy_until``)
    in the loop's time base, but every transfer's DURATION is the copy's
    measured CUDA-event time instead of ``transfer_time(bytes, link)``.

The B200 engine itself (engine.DecodeEngine) does not go through this seam:
it runs the same decisions ahead of the GPU and overlaps copies with real
compute; the seam exists so a user of the reference can keep its loop and
swap in hardware transfers.
"""

from __future__ import annotations

from dataclasses import dataclass
from types import SimpleNamespace

import numpy as np
import torch

from . import _C
from .control import BlockAllocator
from .trace import OutOfMemory


class B200GpuState:
    """``GpuState`` duck type with physical blocks (one stage's pool)."""

    def __init__(self, stage_id: int, total_blocks: int, free_blocks: int, allocator: BlockAllocator = None):
        self.stage_id = stage_id
        self.total_blocks = total_blocks
        self.free_blocks = free_blocks
        self.resident_blocks = {}
        self.alloc = allocator if allocator is not None else BlockAllocator(total_blocks, 0)

    def seed(self, rid, blocks: int):
        """Initial residency (the reference fills ``resident_blocks`` directly)."""
        self.resident_blocks[rid] = blocks
        self.alloc.assign(rid, blocks)

    def allocate(self, rid, blocks: int):
        if blocks > self.free_blocks:
            raise OutOfMemory(f"request {rid} needs {blocks} blocks, only {self.free_blocks} free")
        self.free_blocks -= blocks
        self.resident_blocks[rid] = self.resident_blocks.get(rid, 0) + blocks
        self.alloc.assign(rid, blocks)

    def grow(self, rid):
        if self.free_blocks < 1:
            raise OutOfMemory(f"no free block for token growth of request {rid}")
        self.free_blocks -= 1
        self.resident_blocks[rid] += 1
        self.alloc.append_block(rid)

    def release(self, rid):
        self.free_blocks += self.resident_blocks.pop(rid, 0)
        self.alloc.release(rid)

    @property
    def used_blocks(self) -> int:
        return self.total_blocks - self.free_blocks

    def blocks_of(self, rid) -> list:
        return list(self.alloc.tables.get(rid, []))


@dataclass
class Dispatch:
    """One link occupancy (the reference's ``DispatchRecord`` fields)."""

    queued_at: float
    start: float
    end: float
    priority: str
    n_bytes: int
    chunks: int
    tag: object


class _Handle:
    def __init__(self, when, n_bytes, chunks, tag, ev0, ev1):
        self.submit_time, self.n_bytes, self.chunks, self.tag = when, n_bytes, chunks, tag
        self.ev0, self.ev1 = ev0, ev1
        self.end_time = None
        self.started_at = None


class B200CopyChannel:
    """``ChannelSim`` duck type over a real CUDA copy stream (one direction)."""

    def __init__(self, direction: str, *, pool: torch.Tensor, replica, slot_of: dict, gpu: B200GpuState,
                 block_bytes: int, priority_enabled: bool = True, name: str = None, staging_bytes: int = 64 << 20):
        assert direction in ("h2d", "d2h")
        self.link = SimpleNamespace(direction=direction, busy_until=0.0)
        self.name = name or direction
        self.priority_enabled = priority_enabled
        self.pool, self.rep, self.slot_of, self.gpu = pool, replica, slot_of, gpu
        self.block_bytes = block_bytes
        dev = pool.device
        lo, hi = torch.cuda.Stream.priority_range()
        self.low = torch.cuda.Stream(device=dev, priority=lo)
        self.high = torch.cuda.Stream(device=dev, priority=hi if priority_enabled else lo)
        self.dev_stage = torch.empty(staging_bytes, dtype=torch.uint8, device=dev)
        self.host_stage = torch.empty(staging_bytes, dtype=torch.uint8).pin_memory()
        self.records = []
        self._pending = []
        self.bytes_moved = 0
        self.prefetched = {}      # rid -> physical blocks the last kv_prefetch wrote

    # -- copies ----------------------------------------------------------------
    def _staged_copy(self, n_bytes: int, stream):
        left = n_bytes
        while left > 0:
            k = min(left, self.dev_stage.numel())
            if self.link.direction == "d2h":
                self.host_stage[:k].copy_(self.dev_stage[:k], non_blocking=True)
            else:
                self.dev_stage[:k].copy_(self.host_stage[:k], non_blocking=True)
            left -= k

    def _prefetch_copy(self, rid):
        blocks = self.gpu.blocks_of(rid)
        bb = self.block_bytes
        base = self.rep.offset(self.slot_of[rid])
        dst = np.asarray([pb * bb for pb in blocks], dtype=np.int64)
        src = np.asarray([base + lb * bb for lb in range(len(blocks))], dtype=np.int64)
        _C.call("pm_copy_pieces", _C.C.c_void_p(self.pool.data_ptr()), _C.C.c_void_p(self.rep.ptr),
                dst.ctypes.data_as(_C.C.c_void_p), src.ctypes.data_as(_C.C.c_void_p), len(blocks), bb,
                _C.C.c_void_p(torch.cuda.current_stream().cuda_stream))
        self.prefetched[rid] = blocks
        return len(blocks) * bb

    def _issue(self, stream, fn):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            ev0.record(stream)
            n = fn()
            ev1.record(stream)
        return ev0, ev1, n

    # -- ChannelSim API ----------------------------------------------------------
    def submit_stream(self, when: float, total_bytes: int, chunk_bytes: int, tag: object = None):
        """Queue a chunked low-priority transfer; the copy is issued now on
        the low-priority stream, its end time resolved by finish_stream()."""
        chunks = -(-int(total_bytes) // int(chunk_bytes)) if total_bytes > 0 else 0
        if isinstance(tag, tuple) and tag and tag[0] == "kv_prefetch" and self.link.direction == "h2d":
            rid = tag[1]
            ev0, ev1, n = self._issue(self.low, lambda: self._prefetch_copy(rid))
        else:
            ev0, ev1, n = self._issue(self.low, lambda: (self._staged_copy(int(total_bytes), self.low),
                                                         int(total_bytes))[1])
        h = _Handle(when, n, chunks, tag, ev0, ev1)
        self.bytes_moved += n
        self._pending.append(h)
        return h

    def _resolve(self, upto=None):
        """Settle pending streams in FIFO order: start = max(submit, link
        busy), end = start + the copy's measured duration."""
        while self._pending:
            h = self._pending[0]
            h.ev1.synchronize()
            dur = h.ev0.elapsed_time(h.ev1) * 1e-3
            start = max(h.submit_time, self.link.busy_until)
            h.started_at, h.end_time = start, start + dur
            self.link.busy_until = h.end_time
            self.records.append(Dispatch(h.submit_time, start, h.end_time, "low", h.n_bytes, h.chunks, h.tag))
            self._pending.pop(0)
            if h is upto:
                break

    def submit_high(self, when: float, n_bytes: int, tag: object = None):
        """High-priority transfer (activation hop): returns (start, end)."""
        if n_bytes <= 0:
            self.records.append(Dispatch(when, when, when, "high", 0, 0, tag))
            return when, when
        if not self.priority_enabled:
            self._resolve()          # FIFO baseline: everything submitted goes first
        ev0, ev1, n = self._issue(self.high, lambda: (self._staged_copy(int(n_bytes), self.high), int(n_bytes))[1])
        ev1.synchronize()
        dur = ev0.elapsed_time(ev1) * 1e-3
        start = max(when, self.link.busy_until) if not self.priority_enabled else when
        end = start + dur
        self.link.busy_until = max(self.link.busy_until, end)
        self.bytes_moved += n
        self.records.append(Dispatch(when, start, end, "high", n, 1, tag))
        return start, end

    def finish_stream(self, handle) -> float:
        if handle.end_time is None:
            self._resolve(upto=handle)
        return handle.end_time

    def drain(self) -> float:
        self._resolve()
        return self.link.busy_until
