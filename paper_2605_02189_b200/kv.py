"""KV offload engine of one pipeline stage: pinned host replica + copy-engine
streams, event-ordered against the compute stream.

Replaces the reference's simulated links (REF = reference
``pkg/src/pipemax``): ``ChannelSim.submit_stream`` prefetch (pipeline_sim.py
:442-450, transfer.py:237-257), the eager decode offload (pipeline_sim.py
:486-490) and ``GpuState`` residency (:121-153).

* Host replica: one contiguous, block-first region per request slot
  ``[max_blocks][16][L_s][2][Hkv][hd]`` bf16 in pinned memory.  It is kept
  complete (every new token is offloaded the step it is produced), so an
  eviction costs no copy -- exactly the reference's invariant
  (scheduler.py:318-321).
* Prefetch (plan t): whole blocks host->HBM on the H2D stream, one DMA per
  run of consecutive physical blocks.  Ordered after the compute step that
  last read the reused blocks and after the offload that last wrote the
  prefetched requests' host copy; the step that first executes them waits on
  it (the stall the reference models at pipeline_sim.py:410-421).
* Offload (step t): the new token's whole-stage KV (one contiguous slot per
  row) HBM->host on the D2H stream right after the step's compute: a gather
  kernel packs the rows into a staging slab, ONE cudaMemcpyAsync moves it to
  pinned host staging and a host function in stream order scatters the rows
  into the replica (pm_offload_gather).  PM_OFFLOAD_MODE=dma: one
  cudaMemcpyAsync per run of contiguous rows (pm_copy_pieces).
  PM_OFFLOAD_MODE=kernel selects the SM-side variant (pm_offload_rows: a kernel
  storing through the mapped replica) for A/B only -- measured at ~1 GB/s
  on B200 (SM stores to mapped host memory), which made C2 4x slower
  (profiles/r2/offload_ab.md).
* The replica is pinned on the GPU's NUMA node (pm_host_alloc_numa).
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _C

# decode offload path: "auto" (below), "gather" (pm_offload_gather: gather kernel -> one DMA ->
# host scatter in stream order), "dma" (pm_copy_pieces: one cudaMemcpyAsync per
# run of contiguous rows), "kernel" (pm_offload_rows, SM stores through the
# mapped replica: ~1 GB/s, A/B only)
OFFLOAD_MODE = os.environ.get("PM_OFFLOAD_MODE", "auto")
# auto: gather when a step offloads at least this much (C2: 18 MB/step -> gather,
# 10.4 vs 9.4 GB/s effective; a C3 stage: 1.5 MB/step -> per-row DMAs, where the
# host function's dispatch latency outweighs the saved copy setups)
GATHER_MIN_BYTES = 8 << 20
if os.environ.get("PM_OFFLOAD_DMA") == "0":
    OFFLOAD_MODE = "kernel"
OFFLOAD_CTAS = int(os.environ.get("PM_OFFLOAD_CTAS", "32"))
STAGE_RING = 4   # gather-offload staging slabs (steps in flight on the D2H stream)
# A/B: lanes at staggered stream priorities (lane 0 first for free SMs) instead of equal ones
LANE_PRIO_STAGGER = os.environ.get("PM_LANE_PRIO", "flat") == "stagger"


def device_numa_node(device=None) -> int:
    """NUMA node of the device's PCIe attachment (-1 unknown)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n = _C.C.c_int(-1)
    _C.call("pm_device_numa_node", dev.index if dev.index is not None else torch.cuda.current_device(),
            _C.C.byref(n))
    return int(n.value)


class HostReplica:
    """Pinned host KV: ``slots`` request regions of ``max_blocks`` blocks, on
    the NUMA node of ``device`` (``numa_node`` overrides; -1 = no binding)."""

    def __init__(self, slots: int, max_blocks: int, block_bytes: int, device=None, numa_node: int = None):
        self.slots, self.max_blocks, self.block_bytes = slots, max_blocks, block_bytes
        self.region_bytes = max_blocks * block_bytes
        self.nbytes = slots * self.region_bytes
        if numa_node is None:   # PM_HOST_NUMA overrides (-1 = no binding; A/B)
            env = os.environ.get("PM_HOST_NUMA")
            numa_node = int(env) if env is not None else device_numa_node(device)
        self.numa_node = numa_node
        ptr = _C.C.c_void_p()
        _C.call("pm_host_alloc_numa", self.nbytes, self.numa_node, _C.C.byref(ptr))
        self.ptr = ptr.value
        d = _C.C.c_void_p()
        _C.call("pm_host_device_ptr", _C.C.c_void_p(self.ptr), _C.C.byref(d))
        self.dev_ptr = d.value

    def offset(self, slot: int, block: int = 0) -> int:
        return slot * self.region_bytes + block * self.block_bytes

    def as_tensor(self):
        """uint8 view (tests / prefill seeding)."""
        import ctypes
        buf = (ctypes.c_uint8 * self.nbytes).from_address(self.ptr)
        return torch.frombuffer(buf, dtype=torch.uint8)

    def close(self):
        if self.ptr:
            torch.cuda.synchronize()   # no copy may still read or write the pages being unpinned
            _C.call("pm_host_free_numa", _C.C.c_void_p(self.ptr), self.nbytes, self.numa_node)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class KvEngine:
    """Copy streams, events and the dependency rules of one stage."""

    def __init__(self, executor, replica: HostReplica, slot_of: dict, device, timing: bool = True,
                 low_priority_copies: bool = True):
        """``low_priority_copies``: compute streams above the KV copy streams
        (REF ChannelSim ``priority_enabled``: two priority lanes); False puts
        every stream at the same (lowest) priority -- one FIFO lane."""
        self.ex, self.rep, self.slot_of = executor, replica, slot_of
        self.dev = device
        lo, hi = torch.cuda.Stream.priority_range()
        self._compute_prio = hi if low_priority_copies else lo
        self.compute = torch.cuda.Stream(device=device, priority=self._compute_prio)
        self.streams = [self.compute]   # one compute stream per lane (micro-batch in flight)
        self.h2d = torch.cuda.Stream(device=device, priority=lo)
        self.d2h = torch.cuda.Stream(device=device, priority=lo)
        self.timing = timing
        self.pool_ptr = executor.pool.data_ptr()
        self.block_bytes = executor.block_bytes
        self.tok_bytes = executor.tok_bytes
        self.last_write = {}        # rid -> step whose offload last wrote its host copy
        self.d2h_done = {}          # step -> event
        self.compute_done = {}      # step -> event
        self.h2d_done = {}          # step -> event (plan t's prefetch)
        self.records = []           # per step timing events
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.block_last_d2h = np.full(executor.pool_blocks, -1, dtype=np.int64)
        # per lane: the last step of that lane whose compute read or wrote each
        # block.  With several lanes (micro-batches in flight on different
        # streams) a block freed by one step and reused by a later one needs an
        # explicit compute -> compute edge to the newest toucher on EVERY other
        # lane (same-lane order is stream order); one array per lane so an
        # older toucher on lane B is not masked by a newer one on lane A.
        self.block_last_compute = [np.full(executor.pool_blocks, -1, dtype=np.int64)]
        self._off_ring = None       # mapped pinned (host, pool) offset pairs of the offload kernel
        self._stage = None          # gather offload: [STAGE_RING] (device slab, pinned host slab)
        self._stage_i = 0

    def _offsets(self, n: int):
        """A mapped pinned int64 [n][2] buffer for this step's offload offsets
        (4-deep ring; a buffer is rewritten only after its kernel finished)."""
        if self._off_ring is None:
            import ctypes
            cap = 2 * self.ex.m_cap
            self._off_ring = []
            for _ in range(4):
                p = _C.C.c_void_p()
                _C.call("pm_host_alloc", cap * 8, _C.C.byref(p))
                d = _C.C.c_void_p()
                _C.call("pm_host_device_ptr", p, _C.C.byref(d))
                arr = np.frombuffer((ctypes.c_int64 * cap).from_address(p.value), dtype=np.int64)
                self._off_ring.append([arr, d.value, None, p.value])
            self._off_i = 0
        slot = self._off_ring[self._off_i % 4]
        self._off_i += 1
        if slot[2] is not None:
            slot[2].synchronize()
        return slot
    def _stage_slot(self):
        """(device slab, pinned host slab) of the gather offload, m_cap rows
        each; slots rotate and are reused in D2H-stream order only."""
        if self._stage is None:
            nb = self.ex.m_cap * self.tok_bytes
            self._stage = []
            for _ in range(STAGE_RING):
                d = torch.empty(nb, dtype=torch.uint8, device=self.dev)
                p = _C.C.c_void_p()
                _C.call("pm_host_alloc", nb, _C.C.byref(p))
                self._stage.append((d, p.value))
        slot = self._stage[self._stage_i % STAGE_RING]
        self._stage_i += 1
        return slot

    def __del__(self):
        try:
            for slot in self._off_ring or ():
                _C.call("pm_host_free", _C.C.c_void_p(slot[3]))
            for _, hp in self._stage or ():
                _C.call("pm_host_free", _C.C.c_void_p(hp))
        except Exception:
            pass

    def reset_phase(self):
        """New decode phase (episode.py): step numbers restart at 0, so the
        per-step event maps and block histories start empty (the caller
        synchronized the device)."""
        self.last_write.clear()
        self.d2h_done.clear()
        self.compute_done.clear()
        self.h2d_done.clear()
        self.block_last_d2h[:] = -1
        for a in self.block_last_compute:
            a[:] = -1

    def load_resident(self, tables: dict):
        """Bulk H2D of resident requests' KV (host replica -> their blocks)
        at the start of a decode phase (REF run_episode's initial-residency
        load, pipeline_sim.py:732-739); returns bytes."""
        bb = self.block_bytes
        dst, src = [], []
        for rid in sorted(tables):
            base = self.rep.offset(self.slot_of[rid])
            for lb, pb in enumerate(tables[rid]):
                dst.append(pb * bb)
                src.append(base + lb * bb)
        if dst:
            d = np.asarray(dst, dtype=np.int64)
            sr = np.asarray(src, dtype=np.int64)
            _C.call("pm_copy_pieces", _C.C.c_void_p(self.pool_ptr), _C.C.c_void_p(self.rep.ptr),
                    d.ctypes.data_as(_C.C.c_void_p), sr.ctypes.data_as(_C.C.c_void_p), len(dst), bb,
                    _C.C.c_void_p(self.h2d.cuda_stream))
        return len(dst) * bb

    def add_lane(self) -> int:
        prio = self._compute_prio
        if LANE_PRIO_STAGGER:   # lane i one priority level below lane i - 1 (still above the copies)
            lo, hi = torch.cuda.Stream.priority_range()
            prio = min(lo, self._compute_prio + len(self.streams)) if hi < lo else self._compute_prio
        self.streams.append(torch.cuda.Stream(device=self.dev, priority=prio))
        self.block_last_compute.append(np.full(self.ex.pool_blocks, -1, dtype=np.int64))
        return len(self.streams) - 1

    def _wait_touchers(self, stream, blocks, skip_lane=None, skip_step=None):
        """``stream`` waits for the newest compute step of every lane (except
        ``skip_lane``, ordered by stream order) that touched ``blocks``."""
        for li, arr in enumerate(self.block_last_compute):
            if li == skip_lane:
                continue
            dep = int(arr[blocks].max())
            ev = self.compute_done.get(dep)
            if ev is not None and dep != skip_step:
                stream.wait_event(ev)

    def _event(self):
        return torch.cuda.Event(enable_timing=self.timing)

    # -- H2D prefetch of plan t ---------------------------------------------------
    def prefetch(self, t: int, work, rec: dict):
        """Issue plan t's host->HBM block copies (REF pipeline_sim.py:442-450)."""
        self.records.append(rec)
        if not work.prefetch:
            self.h2d_done[t] = None
            return
        bb = self.block_bytes
        dst, src, targets = [], [], set()
        for rid, blocks, _n in work.prefetch:
            base = self.rep.offset(self.slot_of[rid])
            for lb, pb in enumerate(blocks):
                dst.append(pb * bb)
                src.append(base + lb * bb)
                targets.add(pb)
        s = self.h2d
        # the reused blocks' last readers on every lane (normally step t-1)
        self._wait_touchers(s, np.fromiter(targets, dtype=np.int64))
        # the host copy must hold the requests' last token, and no offload may
        # still be reading a block this copy overwrites
        dep = max((self.last_write.get(rid, -1) for rid, _, _ in work.prefetch), default=-1)
        dep = max(dep, int(self.block_last_d2h[list(targets)].max()))
        ev = self.d2h_done.get(dep)
        if ev is not None:
            s.wait_event(ev)
        with torch.cuda.stream(s):
            if self.timing:
                rec["h2d_start"] = self._event()
                rec["h2d_start"].record(s)
            n = len(dst)
            d = np.asarray(dst, dtype=np.int64)
            sr = np.asarray(src, dtype=np.int64)
            _C.call("pm_copy_pieces", _C.C.c_void_p(self.pool_ptr), _C.C.c_void_p(self.rep.ptr),
                    d.ctypes.data_as(_C.C.c_void_p), sr.ctypes.data_as(_C.C.c_void_p), n, bb,
                    _C.C.c_void_p(s.cuda_stream))
            done = self._event()
            done.record(s)
        rec["h2d_end"] = done
        rec["h2d_bytes"] = len(dst) * bb
        self.h2d_bytes += len(dst) * bb
        self.h2d_done[t] = done

    # -- compute ordering -----------------------------------------------------------
    def before_compute(self, t: int, work, rec: dict):
        s = rec.get("stream", self.compute)
        if self.timing:
            rec["ready"] = self._event()
            rec["ready"].record(s)
        ev = self.h2d_done.get(t - 1)
        if ev is not None:
            s.wait_event(ev)              # batch i's newest members arrived with plan t-1
        if rec.get("serialize"):
            ev = self.compute_done.get(t - 1)
            if ev is not None:
                s.wait_event(ev)
        # blocks this step touches that another lane's step touched last
        used = rec.get("used_blocks")
        if used is not None and len(used):
            lane = rec.get("lane", 0)
            self._wait_touchers(s, used, skip_lane=lane, skip_step=t)
            self.block_last_compute[lane][used] = t
        # a growth block handed out this step may still be read by an offload
        grow = [work.tables[r][p // 16] for r, p in zip(work.rows, work.positions) if p % 16 == 0]
        if grow:
            dep = int(self.block_last_d2h[grow].max())
            ev = self.d2h_done.get(dep)
            if ev is not None:
                s.wait_event(ev)
        if self.timing:
            rec["start"] = self._event()
            rec["start"].record(s)

    def after_compute(self, t: int, rec: dict):
        done = self._event()
        done.record(rec.get("stream", self.compute))
        rec["end"] = done
        self.compute_done[t] = done

    # -- D2H offload of step t --------------------------------------------------------
    def offload(self, t: int, work, rec: dict):
        """Eager offload of the step's new KV (REF pipeline_sim.py:486-490)."""
        rows = work.offload_rows
        if not rows:
            self.d2h_done[t] = None
            return
        tb, bb = self.tok_bytes, self.block_bytes
        src, dst = [], []
        for ix in rows:
            rid, pos = work.rows[ix], work.positions[ix]
            blk = work.tables[rid][pos // 16]
            src.append(blk * bb + (pos % 16) * tb)
            dst.append(self.rep.offset(self.slot_of[rid]) + pos * tb)
            self.last_write[rid] = t
            self.block_last_d2h[blk] = t
        s = self.d2h
        s.wait_event(self.compute_done[t])
        with torch.cuda.stream(s):
            if self.timing:
                rec["d2h_start"] = self._event()
                rec["d2h_start"].record(s)
            mode = OFFLOAD_MODE
            if mode == "auto":   # one gathered DMA pays off for big steps; per-row DMAs for small ones
                mode = "gather" if len(rows) * tb >= GATHER_MIN_BYTES else "dma"
            if mode == "gather":
                d = np.asarray(dst, dtype=np.int64)
                sr = np.asarray(src, dtype=np.int64)
                dslab, hslab = self._stage_slot()
                _C.call("pm_offload_gather", _C.C.c_void_p(self.rep.ptr), _C.C.c_void_p(self.pool_ptr),
                        d.ctypes.data_as(_C.C.c_void_p), sr.ctypes.data_as(_C.C.c_void_p), len(rows), tb,
                        _C.C.c_void_p(dslab.data_ptr()), _C.C.c_void_p(hslab), _C.C.c_void_p(s.cuda_stream))
            elif mode == "dma":
                d = np.asarray(dst, dtype=np.int64)
                sr = np.asarray(src, dtype=np.int64)
                _C.call("pm_copy_pieces", _C.C.c_void_p(self.rep.ptr), _C.C.c_void_p(self.pool_ptr),
                        d.ctypes.data_as(_C.C.c_void_p), sr.ctypes.data_as(_C.C.c_void_p), len(rows), tb,
                        _C.C.c_void_p(s.cuda_stream))
            else:
                slot = self._offsets(len(rows))
                slot[0][0:2 * len(rows):2] = dst
                slot[0][1:2 * len(rows):2] = src
                _C.call("pm_offload_rows", _C.C.c_void_p(self.rep.dev_ptr), _C.C.c_void_p(self.pool_ptr),
                        _C.C.c_void_p(slot[1]), len(rows), tb, OFFLOAD_CTAS, _C.C.c_void_p(s.cuda_stream))
                ev = torch.cuda.Event()
                ev.record(s)
                slot[2] = ev
            done = self._event()
            done.record(s)
        rec["d2h_end"] = done
        rec["d2h_bytes"] = len(rows) * tb
        self.d2h_bytes += len(rows) * tb
        self.d2h_done[t] = done

    # -- accounting ---------------------------------------------------------------------
    def timings(self):
        """(stall_s, h2d_busy_s, d2h_busy_s, compute_s) from the recorded events."""
        stall = h2d = d2h = comp = 0.0
        for rec in self.records:
            if "ready" in rec and "start" in rec:
                stall += rec["ready"].elapsed_time(rec["start"]) * 1e-3
            if "h2d_start" in rec:
                h2d += rec["h2d_start"].elapsed_time(rec["h2d_end"]) * 1e-3
            if "d2h_start" in rec:
                d2h += rec["d2h_start"].elapsed_time(rec["d2h_end"]) * 1e-3
            if "start" in rec and "end" in rec:
                comp += rec["start"].elapsed_time(rec["end"]) * 1e-3
        return stall, h2d, d2h, comp
