"""Host control loop of the B200 decode engine: one call per rotation step.

This is the bookkeeping half of the reference's ``_DecodeEngine.run``
(REF = reference ``pkg/src/pipemax/pipeline_sim.py``, :386-543) with the
simulated clock removed.  Because the reference's decisions never read time,
the loop can run a whole iteration's accounting -- plan, commit, block
mirroring, token bump, completions, block growth with growth-relief
eviction -- BEFORE the GPU executes that step, and hand the executor a
``StepWork`` record that says exactly which requests run, which blocks to
copy in, which slots to offload and which blocks to free.

Physical block ids are assigned here too (``BlockAllocator``): the
reference only pins block COUNTS (``GpuState``), which this loop mirrors in
the reference's exact order so the counts can be checked against golden
streams from the reference itself.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import scheduler as sched
from .model_core import ClusterConfig, EstimatorParams, blocks_for_tokens, capacity_blocks
from .trace import EpisodeMetrics, GpuState, OutOfMemory


class BlockAllocator:
    """Deterministic physical allocator for one stage's block pool.

    ``capacity`` = ``capacity_blocks(cfg)`` accounted blocks plus ``spare``
    extra physical blocks.  The spares absorb the one-step skew between when
    the reference ACCOUNTS a request's new block (iteration end, REF :515-524)
    and when the GPU physically needs it (the step's KV-append writes the new
    token at step start); they also hold the final token of a request that
    completes this step (the reference never allocates that block).  Free ids
    are handed out lowest-first so block tables are reproducible.
    """

    def __init__(self, capacity: int, spare: int):
        import heapq
        self._heapq = heapq
        self.total = capacity + spare
        self._free = list(range(self.total))
        heapq.heapify(self._free)
        self.tables = {}  # rid -> list of physical block ids (logical order)

    @property
    def free_count(self) -> int:
        return len(self._free)

    def take(self) -> int:
        if not self._free:
            raise OutOfMemory("physical block pool exhausted")
        return self._heapq.heappop(self._free)

    def assign(self, rid, n_blocks: int) -> list:
        blocks = [self.take() for _ in range(n_blocks)]
        self.tables.setdefault(rid, []).extend(blocks)
        return blocks

    def append_block(self, rid) -> int:
        b = self.take()
        self.tables.setdefault(rid, []).append(b)
        return b

    def release(self, rid) -> list:
        blocks = self.tables.pop(rid, [])
        for b in blocks:
            self._heapq.heappush(self._free, b)
        return blocks


@dataclass
class StepWork:
    """Everything the stage executors need for rotation step ``t``.

    Rows of the micro-batch are in ascending request id (the canonical order,
    SURVEY.md A.6).  ``positions[r]`` is the cache position the step's input
    token is written to (= prefix length before the step); ``slot_blocks`` /
    ``slot_offsets`` locate that position physically.
    """

    plan: sched.StepPlan
    rows: list                       # exec request ids, ascending
    positions: list                  # per row: prefix length before the step
    prefetch: list                   # [(rid, [phys blocks], n_tokens)] ascending rid
    evicted: list                    # plan evictions (blocks released at commit)
    completed: list                  # rids finishing this step
    relief_evicted: list             # growth-relief victims (REF :364-384)
    offload_rows: list               # row indices whose new KV must reach the host
    released_blocks_end: list        # physical blocks freed at iteration end
    tables: dict                     # rid -> physical block list valid during the step
    predicted_seconds: float = 0.0
    batch_tokens: int = 0


def _note_resident(metrics, resident_tokens, capacity_tokens):
    metrics.max_resident_tokens = max(metrics.max_resident_tokens, resident_tokens)
    frac = resident_tokens / capacity_tokens if capacity_tokens else 0.0
    metrics.max_kv_capacity_fraction = max(metrics.max_kv_capacity_fraction, frac)


class DecodeControl:
    """The replicated control plane: every pipeline rank owns one and they
    all produce the same ``StepWork`` sequence.

    ``requests`` maps id -> ``Request`` (``generated`` is advanced in place,
    as the reference does).  ``mode``/``quota_tokens`` select the prefetch
    policy exactly like the reference's ``_plan_step``.
    """

    def __init__(self, state: sched.SchedulerState, cfg: ClusterConfig, params: EstimatorParams,
                 requests: dict, *, mode: str = "dynamic", quota_tokens: int = 0,
                 spare_blocks: int = None, metrics: EpisodeMetrics = None):
        self.state = state
        self.cfg = cfg
        self.params = params
        self.requests = requests
        self.mode = mode
        self.quota = quota_tokens
        self.metrics = metrics or EpisodeMetrics()
        bs = cfg.block_size
        state.configure_blocks(bs)
        cap = capacity_blocks(cfg)
        # reference block counts (REF :561-565)
        self.gpu = GpuState(stage_id=0, total_blocks=cap, free_blocks=cap - state.resident_blocks())
        for rid in state.gpu_resident:
            self.gpu.resident_blocks[rid] = blocks_for_tokens(state.lengths[rid], bs)
        if spare_blocks is None:
            # at most one in-flight growth block per row of the largest
            # possible micro-batch, i.e. per live request
            spare_blocks = max(1, len(state.lengths))
        self.spare_blocks = spare_blocks
        self.alloc = BlockAllocator(cap, spare_blocks)
        for rid in sorted(state.gpu_resident):
            self.alloc.assign(rid, blocks_for_tokens(state.lengths[rid], bs))
        self.resident_tokens = sum(state.lengths[r] for r in state.gpu_resident)
        self.capacity_tokens = cap * bs
        self.live_tokens = sum(state.lengths.values())
        self.pool_was_empty = not state.cpu_pool
        self.finished = False

    # -- reference engine helpers (REF :364-384) ------------------------------

    def _relief_victim(self, batch_idx, growing):
        for rid in sorted(self.state.batches[batch_idx]):
            if rid != growing and rid in self.state.gpu_resident:
                return rid
        return None

    def _evict_for_relief(self, rid):
        st = self.state
        idx = st._batch_of.pop(rid)
        st.batches[idx].remove(rid)
        st._batch_tokens[idx] -= st.lengths[rid]
        st.gpu_resident.remove(rid)
        st._resident_blocks -= blocks_for_tokens(st.lengths[rid], self.cfg.block_size)
        st._pool_add(rid)
        self.gpu.release(rid)
        self.resident_tokens -= st.lengths[rid]
        self.metrics.growth_relief_evictions += 1

    # -- one rotation step ----------------------------------------------------

    def step(self):
        """Advance one iteration; returns ``StepWork`` or None when done
        (same stop rules as REF :392-407)."""
        st, cfg, bs = self.state, self.cfg, self.cfg.block_size
        if self.finished or not st.lengths:
            self.finished = True
            return None
        idle = not any(st.batches)
        if idle and (self.mode == "none" or not st.cpu_pool):
            self.finished = True
            return None
        try:
            plan = sched._plan_step(st, self.params, cfg, mode=self.mode, quota_tokens=self.quota)
        except sched.EmptySystem:
            self.finished = True
            return None
        if not plan.exec_batch and not plan.prefetch_set and idle:
            self.finished = True
            return None

        i = plan.exec_batch_index
        rows = sorted(plan.exec_batch)
        positions = [st.lengths[r] for r in rows]
        batch_tokens = st.batch_tokens(i)

        # commit + mirror into block counts and physical blocks (REF :430-440)
        sched.commit_plan(st, plan, cfg)
        for rid in plan.evictions:
            self.gpu.release(rid)
            self.alloc.release(rid)
            self.resident_tokens -= st.lengths[rid]
        prefetch = []
        for rid in sorted(plan.prefetch_set):
            nb = blocks_for_tokens(st.lengths[rid], bs)
            self.gpu.allocate(rid, nb)
            prefetch.append((rid, self.alloc.assign(rid, nb), st.lengths[rid]))
            self.resident_tokens += st.lengths[rid]
        self.pool_was_empty = not st.cpu_pool
        _note_resident(self.metrics, self.resident_tokens, self.capacity_tokens)

        # physical growth for this step's new token happens NOW (the
        # KV-append writes it); the reference accounts it at iteration end.
        for r, pos in zip(rows, positions):
            if pos % bs == 0:
                self.alloc.append_block(r)
        tables = {r: list(self.alloc.tables[r]) for r in rows}

        # iteration end (REF :494-525)
        completed, crossings = [], []
        for rid in rows:
            crossed = st.bump_generated(rid)
            self.resident_tokens += 1
            self.live_tokens += 1
            req = self.requests[rid]
            req.generated += 1
            self.metrics.total_tokens_generated += 1
            if req.done:
                completed.append(rid)
            elif crossed:
                crossings.append(rid)
        released = []
        for rid in completed:
            self.resident_tokens -= st.lengths[rid]
            self.live_tokens -= st.lengths[rid]
            st.remove_request(rid)
            self.gpu.release(rid)
            released += self.alloc.release(rid)
            self.metrics.completed_requests += 1
        relief = []
        for rid in crossings:
            if rid not in st.gpu_resident:
                continue
            while self.gpu.free_blocks < 1:
                victim = self._relief_victim(i, rid)
                if victim is None:
                    raise OutOfMemory(f"no block for growth of request {rid} and no victim")
                self._evict_for_relief(victim)
                released += self.alloc.release(victim)
                relief.append(victim)
            self.gpu.grow(rid)
        _note_resident(self.metrics, self.resident_tokens, self.capacity_tokens)

        done = set(completed)
        offload_rows = [ix for ix, r in enumerate(rows) if r not in done]
        m = self.metrics
        m.exec_predicted_series.append(plan.predicted_exec_seconds)
        m.max_active_batch_tokens = max(m.max_active_batch_tokens, batch_tokens)
        if plan.steady:
            if m.steady_iteration is None:
                m.steady_iteration = m.iterations
            denom = plan.residual_tokens + plan.prefetch_tokens
            if denom > 0 and not self.pool_was_empty:
                m.prefetched_token_fraction.append(plan.prefetch_tokens / denom)
        m.iterations += 1
        return StepWork(plan=plan, rows=rows, positions=positions, prefetch=prefetch,
                        evicted=list(plan.evictions), completed=completed,
                        relief_evicted=relief, offload_rows=offload_rows,
                        released_blocks_end=released, tables=tables,
                        predicted_seconds=plan.predicted_exec_seconds,
                        batch_tokens=batch_tokens)
