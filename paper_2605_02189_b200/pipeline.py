"""Multi-GPU pipeline: one rank per stage, NCCL P2P between stages.

Replaces the reference's simulated activation hop (``d2h.submit_high`` +
``h2d.submit_high``, REF pipeline_sim.py:455-459) with real device-to-device
transfers, and makes the last->first token return explicit (the reference
leaves it implicit, :411, :484).

Every rank runs the same ``DecodeControl`` (deterministic, so the plan stream
is replicated without communication; ``plan_digest`` lets a debug run compare
it across ranks).  Per rotation step t on stage s:

  * s > 0  : receive the micro-batch's activations [M, d] from s-1;
  * s == 0 : before step t, receive greedy ids of every earlier step whose rows
             appear in step t (in step order -- normally just step t-m), and
             scatter them into the token table by slot;
  * forward its layers (StageExecutor), KV prefetch/offload on its own copy
    streams (KvEngine, same rules as the single-process engine);
  * s < last: send activations to s+1;  s == last: send ids to stage 0.

The schedule is written against a small ``Link`` interface so the same code
runs on NCCL/CUDA and on gloo/CPU (tests/test_pipeline_gloo.py drives it with a
CPU stand-in executor).
"""

from __future__ import annotations

import hashlib

import torch
import torch.distributed as dist

from .control import DecodeControl


def plan_digest(work) -> str:
    p = work.plan
    key = (p.t, tuple(work.rows), tuple(sorted(p.prefetch_set)), p.evictions, tuple(work.completed),
           tuple(work.relief_evicted))
    return hashlib.sha1(repr(key).encode()).hexdigest()[:16]


class Link:
    """torch.distributed P2P with a 2-deep send ring (a send buffer is reused
    only after its previous send completed)."""

    def __init__(self, rank: int, world: int, make_buf):
        self.rank, self.world = rank, world
        self.make_buf = make_buf
        self.ring = [None, None]
        self.pending = [None, None]
        self.k = 0

    def send(self, src: torch.Tensor, dst: int):
        k = self.k % 2
        self.k += 1
        if self.pending[k] is not None:
            self.pending[k].wait()
        if self.ring[k] is None or self.ring[k].numel() < src.numel() or self.ring[k].dtype != src.dtype:
            self.ring[k] = self.make_buf(src)
        buf = self.ring[k][: src.numel()].view_as(src)
        buf.copy_(src)
        self.pending[k] = dist.isend(buf, dst)

    @staticmethod
    def recv(into: torch.Tensor, src: int):
        dist.irecv(into, src).wait()

    def drain(self):
        for w in self.pending:
            if w is not None:
                w.wait()


class PipelineRank:
    """One pipeline stage.  ``executor`` is a StageExecutor (or a stand-in
    with ``resid``, ``out_ids``, ``tok_table``, ``forward(M)``), ``kv`` a
    KvEngine or None."""

    def __init__(self, control: DecodeControl, executor, slot_of: dict, *, rank: int, world: int, kv=None,
                 upload_meta=None, stream=None, bucket=lambda m: m):
        self.control, self.ex, self.kv = control, executor, kv
        self.slot_of = slot_of
        self.rank, self.world = rank, world
        self.first, self.last = rank == 0, rank == world - 1
        self.upload_meta = upload_meta
        self.stream = stream
        self.bucket = bucket
        dev = executor.resid.device
        self.link = Link(rank, world, lambda t: torch.empty(t.numel() * 2, dtype=t.dtype, device=dev))
        self.t = 0
        self.last_step = {}       # rid -> last step it executed (stage 0's token dependency)
        self.ids_rows = {}        # step -> rows whose ids are outstanding (stage 0)
        self.ids_next = 0         # next step whose ids stage 0 will receive
        self.digests = []

    def _receive_ids_until(self, upto: int):
        # stage 0: receive ids of steps ids_next..upto in order, scatter by slot
        ex = self.ex
        while self.ids_next <= upto:
            rows = self.ids_rows.pop(self.ids_next)
            if rows:
                buf = torch.empty(self.bucket(len(rows)), dtype=torch.int32, device=ex.tok_table.device)
                self.link.recv(buf, self.world - 1)
                idx = torch.tensor([self.slot_of[r] for r in rows], dtype=torch.long, device=buf.device)
                ex.tok_table[idx] = buf[: len(rows)]
            self.ids_next += 1

    def step(self):
        work = self.control.step()
        if work is None:
            return None
        t = self.t
        self.digests.append(plan_digest(work))
        M = len(work.rows)
        Mb = self.bucket(M)
        ex = self.ex
        rec = {"t": t, "M": M}
        if self.kv is not None:
            self.kv.prefetch(t, work, rec)
        ctx = torch.cuda.stream(self.stream) if self.stream is not None else _Null()
        with ctx:
            if self.upload_meta is not None:
                self.upload_meta(work.rows, work.positions, work.tables)
            if self.kv is not None:
                self.kv.before_compute(t, work, rec)
            if self.first and self.world > 1:
                need = max((self.last_step.get(r, -1) for r in work.rows), default=-1)
                self._receive_ids_until(need)
            if M > 0:  # empty steps move nothing on any rank (the plan stream is replicated)
                if not self.first:
                    self.link.recv(ex.resid[:Mb], self.rank - 1)
                ex.forward(Mb)
                if not self.last:
                    self.link.send(ex.resid[:Mb], self.rank + 1)
                elif self.world > 1:
                    self.link.send(ex.out_ids[:Mb], 0)
            if self.kv is not None:
                self.kv.after_compute(t, rec)
                self.kv.offload(t, work, rec)
        if self.first and self.world > 1:
            self.ids_rows[t] = list(work.rows)
        for r in work.rows:
            self.last_step[r] = t
        self.t += 1
        return work

    def finish(self):
        """Drain outstanding sends/receives so every rank ends cleanly."""
        if self.first and self.world > 1:
            self._receive_ids_until(self.t - 1)
        self.link.drain()


class PipelineEngine:
    """One pipeline rank of a multi-GPU run (torchrun, NCCL): the stage this
    rank owns (layers, KV pool, host replica, copy streams) driven by the
    replicated control plane and the P2P schedule of ``PipelineRank``."""

    def __init__(self, spec, state, cfg, params, requests, *, rank, world, device, seed=0, graphs=True, **kw):
        from .engine import DecodeEngine
        self.eng = DecodeEngine(spec, state, cfg, params, requests, pp=world, device=device, seed=seed,
                                graphs=graphs, local_stages=[rank], **kw)
        ex, kv = self.eng.stages[0]
        self.ex, self.kv = ex, kv
        eng = self.eng

        class _Fwd:  # forward through the stage's CUDA graphs
            resid, out_ids, tok_table = ex.resid, ex.out_ids, ex.tok_table

            def forward(self_, M):
                ex.run(M, kv.compute, graphs=eng.graphs)

        self.pr = PipelineRank(eng.control, _Fwd(), eng.slot_of, rank=rank, world=world, kv=kv,
                               upload_meta=lambda rows, pos, tab: eng._upload_meta(rows, pos, tab, stream=kv.compute),
                               stream=kv.compute, bucket=eng.bucket)

    @property
    def metrics(self):
        return self.eng.metrics

    def step(self):
        return self.pr.step()

    def finish(self):
        self.pr.finish()


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
