"""Diagnostic: the two-rank pipeline vs the single-process PP=2 engine on the
test scenario -- dumps stage inputs/outputs of the first steps."""
import os
import socket
import sys

import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_pipeline_gpu import _scenario  # noqa: E402


def worker(rank, port, steps):
    from paper_2605_02189_b200.pipeline import PipelineEngine, make_groups
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    spec, st, cfg, params, reqs = _scenario()
    peng = PipelineEngine(spec, st, cfg, params, reqs, rank=rank, world=2, device="cuda:0", kv_init="random", seed=5,
                          transport="staged", groups=make_groups(2))
    ex = peng.ex
    out = {"pool": ex.pool.float().sum().item(), "tok": ex.tok_table.clone().cpu()}
    for n in range(steps):
        w = peng.step()
        torch.cuda.synchronize()
        out[n] = dict(rows=w.rows, resid=ex.resid[:len(w.rows)].clone().cpu(), ids=ex.out_ids[:len(w.rows)].clone().cpu(),
                      bt=ex.block_table[:len(w.rows)].clone().cpu(), pos=ex.positions[:len(w.rows)].clone().cpu(),
                      sl=ex.seq_lens[:len(w.rows)].clone().cpu())
    torch.save(out, f"gpurun_out/diag_rank{rank}.pt")
    peng.finish()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    from paper_2605_02189_b200.engine import DecodeEngine
    steps = 3
    spec, st, cfg, params, reqs = _scenario()
    ref = DecodeEngine(spec, st, cfg, params, reqs, pp=2, kv_init="random", seed=5, graphs=True)
    ref_out = {s: {"pool": ex.pool.float().sum().item(), "tok": ex.tok_table.clone().cpu()} for s, (ex, _) in enumerate(ref.stages)}
    for n in range(steps):
        w = ref.step()
        torch.cuda.synchronize()
        for s, (ex, _) in enumerate(ref.stages):
            ref_out[s][n] = dict(rows=w.rows, resid=ex.resid[:len(w.rows)].clone().cpu(),
                                 ids=ex.out_ids[:len(w.rows)].clone().cpu(), bt=ex.block_table[:len(w.rows)].clone().cpu(),
                                 pos=ex.positions[:len(w.rows)].clone().cpu(), sl=ex.seq_lens[:len(w.rows)].clone().cpu())
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(worker, args=(port, steps), nprocs=2)
    for rank in range(2):
        got = torch.load(f"gpurun_out/diag_rank{rank}.pt")
        want = ref_out[rank]
        print(f"rank {rank}: pool sum {got['pool']} vs {want['pool']}; tok table equal {torch.equal(got['tok'], want['tok'])}")
        for n in range(steps):
            g, r = got[n], want[n]
            print(f"  step {n} rows {g['rows']} {r['rows']} resid max|d| {(g['resid'] - r['resid']).abs().max().item():.3g} "
                  f"ids {g['ids'].tolist()} {r['ids'].tolist()} bt_eq {torch.equal(g['bt'], r['bt'])} "
                  f"pos_eq {torch.equal(g['pos'], r['pos'])} sl_eq {torch.equal(g['sl'], r['sl'])}")
            if rank == 1:
                print("   resid rows diff per row", (g['resid'] - r['resid']).abs().amax(1).tolist())
