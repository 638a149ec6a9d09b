"""Multi-GPU pipeline: one rank per stage, P2P between stages.

Replaces the reference's simulated activation hop (``d2h.submit_high`` +
``h2d.submit_high``, REF pipeline_sim.py:455-459) with real device-to-device
transfers, and makes the last->first token return explicit (the reference
leaves it implicit, :411, :484).

Every rank runs the same ``DecodeControl`` (deterministic, so the plan stream
is replicated without communication; ``plan_digest`` lets a debug run compare
it across ranks).  Per rotation step t on stage s (REF stage walk
pipeline_sim.py:452-484):

  * s > 0  : receive the micro-batch's activations from s-1 (bf16 on the wire,
             pm_hop_unpack into the fp32 residual);
  * s == 0 : before step t, receive greedy ids of every earlier step whose rows
             appear in step t (in step order -- normally just step t-m), and
             scatter them into the token table by slot (pm_scatter_tokens; the
             slots are read from mapped pinned memory -- no copy, no host sync);
  * forward its layers (StageExecutor), KV prefetch/offload on its own copy
             streams (KvEngine, same rules as the single-process engine);
  * s < last: pack (pm_hop_pack) and send activations to s+1;
    s == last: send ids to stage 0.

The two directions use two process groups (``groups``): with NCCL each group
is its own communicator with its own stream, so the forward activation chain
and the backward id return never order against each other -- a rank's send to
s+1 can never wait behind its receive from the last stage (the deadlock a
single communicator allows once messages exceed NCCL's buffering).

Transports: ``nccl`` (CUDA tensors straight to NCCL), ``staged`` (CUDA
tensors through pinned host memory over gloo -- two processes sharing one GPU,
tests/test_pipeline_gpu.py), and plain CPU tensors over gloo
(tests/test_pipeline_gloo.py drives the schedule with a CPU stand-in stage).
"""

from __future__ import annotations

import hashlib

import torch
import torch.distributed as dist

from . import _C
from .control import DecodeControl


def plan_digest(work) -> str:
    p = work.plan
    key = (p.t, tuple(work.rows), tuple(sorted(p.prefetch_set)), p.evictions, tuple(work.completed),
           tuple(work.relief_evicted))
    return hashlib.sha1(repr(key).encode()).hexdigest()[:16]


class Link:
    """P2P in one direction on one process group, with a 2-deep send ring (a
    send buffer is reused only after its previous send completed).
    ``staged``: CUDA tensors go through pinned host memory (gloo)."""

    def __init__(self, group=None, staged: bool = False):
        self.group, self.staged = group, staged
        self.ring = [None, None]
        self.host = [None, None]
        self.pending = [None, None]
        self.k = 0
        self.rbuf = None

    def send_buffer(self, numel: int, dtype, device) -> torch.Tensor:
        """The next ring slot (waits for its previous send): fill it, then send_filled()."""
        k = self.k % 2
        if self.pending[k] is not None:
            self.pending[k].wait()
            self.pending[k] = None
        if self.ring[k] is None or self.ring[k].numel() < numel or self.ring[k].dtype != dtype:
            self.ring[k] = torch.empty(2 * numel, dtype=dtype, device=device)
        return self.ring[k][:numel]

    def send_filled(self, buf: torch.Tensor, dst: int):
        k = self.k % 2
        self.k += 1
        if self.staged and buf.is_cuda:
            if self.host[k] is None or self.host[k].numel() < buf.numel() or self.host[k].dtype != buf.dtype:
                self.host[k] = torch.empty(2 * buf.numel(), dtype=buf.dtype).pin_memory()
            h = self.host[k][: buf.numel()]
            h.copy_(buf)   # synchronous D2H: the send reads host memory
            buf = h
        self.pending[k] = dist.isend(buf, dst, group=self.group)

    def send(self, src: torch.Tensor, dst: int):
        buf = self.send_buffer(src.numel(), src.dtype, src.device)
        buf.copy_(src.reshape(-1))
        self.send_filled(buf, dst)

    def recv(self, into: torch.Tensor, src: int):
        if self.staged and into.is_cuda:
            if self.rbuf is None or self.rbuf.numel() < into.numel() or self.rbuf.dtype != into.dtype:
                self.rbuf = torch.empty(2 * into.numel(), dtype=into.dtype).pin_memory()
            h = self.rbuf[: into.numel()].view_as(into)
            dist.irecv(h, src, group=self.group).wait()
            into.copy_(h)   # synchronous: the host buffer is reused by the next receive
            return
        dist.irecv(into, src, group=self.group).wait()   # NCCL: stream-ordered, no host block

    def drain(self):
        for i, w in enumerate(self.pending):
            if w is not None:
                w.wait()
                self.pending[i] = None


class _SlotRing:
    """Mapped pinned int32 buffers for the slots of returned ids (stage 0):
    the scatter kernel reads them over PCIe; a buffer is rewritten only after
    the kernel that read it completed."""

    def __init__(self, n: int, depth: int = 4):
        import ctypes
        self.bufs, self.dev, self.raw, self.events = [], [], [], [None] * depth
        for _ in range(depth):
            p = _C.C.c_void_p()
            _C.call("pm_host_alloc", n * 4, _C.C.byref(p))
            d = _C.C.c_void_p()
            _C.call("pm_host_device_ptr", p, _C.C.byref(d))
            self.bufs.append(torch.frombuffer((ctypes.c_int32 * n).from_address(p.value), dtype=torch.int32))
            self.dev.append(d.value)
            self.raw.append(p.value)
        self.i = 0

    def next(self):
        k = self.i % len(self.bufs)
        self.i += 1
        if self.events[k] is not None:
            self.events[k].synchronize()
        return k

    def __del__(self):
        try:
            for p in self.raw:
                _C.call("pm_host_free", _C.C.c_void_p(p))
        except Exception:
            pass


class PipelineRank:
    """One pipeline stage.  ``executor`` is a StageExecutor (or a stand-in
    with ``resid``, ``out_ids``, ``tok_table``, ``forward(M)``), ``kv`` a
    KvEngine or None.  ``groups`` = (activation group, id-return group);
    ``staged``: CUDA tensors over gloo through pinned host memory."""

    def __init__(self, control: DecodeControl, executor, slot_of: dict, *, rank: int, world: int, kv=None,
                 upload_meta=None, stream=None, bucket=lambda m: m, groups=(None, None), staged: bool = False):
        self.control, self.ex, self.kv = control, executor, kv
        self.slot_of = slot_of
        self.rank, self.world = rank, world
        self.first, self.last = rank == 0, rank == world - 1
        self.upload_meta = upload_meta
        self.stream = stream
        self.bucket = bucket
        self.act = Link(groups[0], staged)
        self.ids = Link(groups[1], staged)
        dev = executor.resid.device
        self.cuda = dev.type == "cuda"
        m_cap = executor.resid.shape[0]
        if self.cuda:
            # the activation hop travels as bf16 (half the bytes of the fp32 residual)
            self.act_rbuf = torch.empty(executor.resid.numel(), dtype=torch.bfloat16, device=dev)
            self.ids_rbuf = torch.empty(m_cap, dtype=torch.int32, device=dev)
            self.slot_ring = _SlotRing(m_cap) if (self.first and world > 1) else None
        self.t = 0
        self.last_step = {}       # rid -> last step it executed (stage 0's token dependency)
        self.ids_rows = {}        # step -> rows whose ids are outstanding (stage 0)
        self.ids_next = 0         # next step whose ids stage 0 will receive
        self.digests = []

    def _cs(self):
        return torch.cuda.current_stream() if self.stream is None else self.stream

    def _receive_ids_until(self, upto: int):
        # stage 0: receive ids of steps ids_next..upto in order, scatter by slot
        ex = self.ex
        while self.ids_next <= upto:
            rows = self.ids_rows.pop(self.ids_next)
            if rows:
                n = self.bucket(len(rows))
                if self.cuda:
                    buf = self.ids_rbuf[:n]
                    self.ids.recv(buf, self.world - 1)
                    k = self.slot_ring.next()
                    self.slot_ring.bufs[k][: len(rows)] = torch.tensor([self.slot_of[r] for r in rows],
                                                                       dtype=torch.int32)
                    st = self._cs()
                    _C.call("pm_scatter_tokens", _C.C.c_void_p(buf.data_ptr()), _C.C.c_void_p(self.slot_ring.dev[k]),
                            len(rows), _C.C.c_void_p(ex.tok_table.data_ptr()), _C.C.c_void_p(st.cuda_stream))
                    ev = torch.cuda.Event()
                    ev.record(st)
                    self.slot_ring.events[k] = ev
                else:   # CPU stand-in stage (schedule tests)
                    buf = torch.empty(n, dtype=torch.int32)
                    self.ids.recv(buf, self.world - 1)
                    ex.tok_table[torch.tensor([self.slot_of[r] for r in rows])] = buf[: len(rows)]
            self.ids_next += 1

    def _recv_act(self, Mb):
        ex = self.ex
        if not self.cuda:
            self.act.recv(ex.resid[:Mb], self.rank - 1)
            return
        n = Mb * ex.resid.shape[1]
        buf = self.act_rbuf[:n]
        self.act.recv(buf, self.rank - 1)
        _C.call("pm_hop_unpack", _C.C.c_void_p(buf.data_ptr()), _C.C.c_void_p(ex.resid.data_ptr()), n,
                _C.C.c_void_p(self._cs().cuda_stream))

    def _send_act(self, Mb):
        ex = self.ex
        if not self.cuda:
            self.act.send(ex.resid[:Mb], self.rank + 1)
            return
        n = Mb * ex.resid.shape[1]
        buf = self.act.send_buffer(n, torch.bfloat16, ex.resid.device)
        _C.call("pm_hop_pack", _C.C.c_void_p(ex.resid.data_ptr()), _C.C.c_void_p(buf.data_ptr()), n,
                _C.C.c_void_p(self._cs().cuda_stream))
        self.act.send_filled(buf, self.rank + 1)

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
                used = self.upload_meta(work.rows, work.positions, work.tables)
                if used is not None:
                    # blocks this step touches: a later prefetch into one of them waits
                    # for this step's compute (without it an H2D copy could overwrite KV
                    # an in-flight step still reads)
                    rec["used_blocks"] = used
            if self.kv is not None:
                self.kv.before_compute(t, work, rec)
            if self.first and self.world > 1:
                need = max((self.last_step.get(r, -1) for r in work.rows), default=-1)
                self._receive_ids_until(need)
            if M > 0:  # empty steps move nothing on any rank (the plan stream is replicated)
                if not self.first:
                    self._recv_act(Mb)
                ex.forward(Mb)
                if not self.last:
                    self._send_act(Mb)
                elif self.world > 1:
                    self.ids.send(ex.out_ids[:Mb], 0)
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
        """Drain outstanding sends/receives so every rank ends cleanly (on the
        stage's stream: a receive must not overwrite the id buffer while the
        previous scatter kernel may still read it)."""
        ctx = torch.cuda.stream(self.stream) if self.stream is not None else _Null()
        with ctx:
            if self.first and self.world > 1:
                self._receive_ids_until(self.t - 1)
            self.act.drain()
            self.ids.drain()


def make_groups(world: int, backend: str = None):
    """The two P2P process groups (activations s -> s+1, ids last -> 0)."""
    ranks = list(range(world))
    return dist.new_group(ranks, backend=backend), dist.new_group(ranks, backend=backend)


class PipelineEngine:
    """One pipeline rank of a multi-GPU run (torchrun, NCCL): the stage this
    rank owns (layers, KV pool, host replica, copy streams) driven by the
    replicated control plane and the P2P schedule of ``PipelineRank``.
    ``transport``: "nccl" (default), or "staged" (gloo through pinned host
    memory, for several ranks sharing one GPU)."""

    def __init__(self, spec, state, cfg, params, requests, *, rank, world, device, seed=0, graphs=True,
                 transport="nccl", groups=None, **kw):
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

        if groups is None and world > 1:
            groups = make_groups(world)
        self.pr = PipelineRank(eng.control, _Fwd(), eng.slot_of, rank=rank, world=world, kv=kv,
                               upload_meta=lambda rows, pos, tab: eng._upload_meta(rows, pos, tab, stream=kv.compute),
                               stream=kv.compute, bucket=eng.bucket, groups=groups or (None, None),
                               staged=transport == "staged")

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
