"""Command-line front end of the B200 decode path:

  python -m paper_2605_02189_b200.cli {decode|prefill|episode|compare|calibrate|report} ...

Mirrors the reference's ``pipemax-sim`` (REF = reference ``pkg/src/pipemax``,
cli.py:1-454) for the subcommands that exist on hardware:

* ``decode``    -- ``run_decode`` on a synthetic BASELINE-shaped workload;
                   writes the trace JSONL and the metrics record (reference
                   schemas, REF pipeline_sim.py:57-96 / 156-216);
* ``prefill``   -- ``run_prefill`` (layer-wise offload); trace JSONL + makespan;
* ``episode``   -- ``run_episode`` (prefill <-> decode switching, episode.py);
* ``compare``   -- the same seeded workload under several policies, CSV of
                   tokens/s, stall and prefetched fraction (REF cli.py:197-230);
* ``calibrate`` -- measured (b, L, seconds) samples of this GPU (the CSV the
                   reference's ``calibrate`` reads) and the fitted estimator
                   JSON (REF cli.py:311-327);
* ``report``    -- the reference's per-iteration decode series from a trace
                   (REF cli.py:362-397, same CSV columns).

Exit codes follow the reference (cli.py:5-6, 443-454): 0 ok, 2 configuration
error, 3 runtime capacity/accounting error.
"""

from __future__ import annotations

import argparse
import csv
import json
import sys


class ConfigError(ValueError):
    pass


def _workload(args):
    from .workloads import decode_workload
    from .models import SPECS
    if args.model not in SPECS:
        raise ConfigError(f"unknown model {args.model!r} (one of {sorted(SPECS)})")
    return decode_workload(args.model, args.requests, args.prompt, args.gen, args.micro_batches, args.pool_frac,
                           args.resident_frac)


def _prompts(spec, reqs, seed):
    import numpy as np
    rng = np.random.default_rng(seed)
    return {r: rng.integers(0, spec.vocab, q.input_len) for r, q in reqs.items()}


def cmd_decode(args) -> int:
    from .engine import run_decode
    spec, state, cfg, params, reqs, desc = _workload(args)
    kw = {}
    if args.prefill:
        kw.update(kv_init="prefill", prompts=_prompts(spec, reqs, args.seed))
    trace, metrics = run_decode(state, cfg, params, None, args.horizon, requests=reqs, seed=args.seed,
                                model=spec, pp=args.pp, **kw)
    trace.to_jsonl(args.trace)
    record = metrics.to_record("dynamic", args.seed)
    with open(args.metrics, "w") as fh:
        json.dump(record, fh, indent=2, sort_keys=True)
        fh.write("\n")
    print(f"{record.get('tokens_per_second', 0.0):.1f} tokens/s over {record.get('iterations', '?')} iterations; "
          f"trace -> {args.trace}, metrics -> {args.metrics}")
    return 0


def cmd_prefill(args) -> int:
    from .prefill import run_prefill
    spec, state, cfg, params, reqs, desc = _workload(args)
    trace, makespan, eng = run_prefill(reqs, _prompts(spec, reqs, args.seed), cfg, params, spec,
                                       staging_pool_requests=args.staging, pp=args.pp)
    trace.to_jsonl(args.trace)
    starts = {(e.payload.get("stage"), e.payload.get("request")): e.time for e in trace.select("stall_start")}
    stall = sum(e.time - starts.get((e.payload.get("stage"), e.payload.get("request")), e.time)
                for e in trace.select("stall_end"))
    print(f"prefill makespan {makespan * 1e3:.3f} ms, offload backpressure stalls {stall * 1e3:.3f} ms; "
          f"trace -> {args.trace}")
    return 0


def cmd_calibrate(args) -> int:
    from .calibrate import calibrate_on_device, params_dict, write_samples_csv
    from .engine import DecodeEngine
    spec, state, cfg, params, reqs, desc = _workload(args)
    eng = DecodeEngine(spec, state, cfg, params, reqs, pp=args.pp, kv_init="random")
    fitted, samples, err = calibrate_on_device(eng, reps=args.reps)
    write_samples_csv(args.samples, samples)
    with open(args.out, "w") as fh:
        json.dump(params_dict(fitted), fh, indent=2, sort_keys=True)
        fh.write("\n")
    print(f"alpha={fitted.alpha:.6e} beta={fitted.beta:.6e} delta={fitted.delta:.6e} "
          f"(max rel fit err {err:.3f}); samples -> {args.samples}")
    return 0


def _episode(args, policy):
    from .episode import B200Backend, run_episode
    from .model_core import Request
    spec, state, cfg, params, reqs, desc = _workload(args)
    if args.host_tokens:
        import dataclasses
        cfg = dataclasses.replace(cfg, cpu_kv_capacity=args.host_tokens * cfg.kv_bytes_per_token)
    fresh = {r: Request(r, q.input_len, q.output_len) for r, q in reqs.items()}
    backend = B200Backend(spec, cfg, params, fresh, _prompts(spec, fresh, args.seed), seed=args.seed)
    m = run_episode(list(fresh.values()), cfg, params, policy=policy, seed=args.seed, backend=backend,
                    rho_hi=args.rho_hi, horizon=args.horizon)
    return m.to_record(policy, args.seed)


def cmd_episode(args) -> int:
    """Prefill <-> decode episode on the GPU (REF run_episode)."""
    record = _episode(args, args.policy)
    with open(args.metrics, "w") as fh:
        json.dump(record, fh, indent=2, sort_keys=True)
        fh.write("\n")
    print(f"{record['tokens_per_second']:.1f} tokens/s, {record['phase_switches']} phase switches, "
          f"{record['completed_requests']} completed; metrics -> {args.metrics}")
    return 0


def cmd_compare(args) -> int:
    """The same seeded workload under several policies (REF cli.py:197-230)."""
    policies = [p.strip() for p in args.policies.split(",") if p.strip()]
    rows = []
    for policy in policies:
        rec = _episode(args, policy)
        rows.append((policy, rec["tokens_per_second"], rec["stall_seconds"], rec["mean_prefetched_token_fraction"]))
    with open(args.out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["policy", "tokens_per_second", "stall_seconds", "prefetched_token_fraction"])
        for r in rows:
            w.writerow([r[0], f"{r[1]:.6f}", f"{r[2]:.6f}", f"{r[3]:.6f}"])
    for r in rows:
        print(f"{r[0]}: {r[1]:.3f} tokens/s")
    return 0


def cmd_report(args) -> int:
    """Per-iteration decode series of stage 0 (REF cli.py:362-397)."""
    rows = []
    try:
        with open(args.trace) as fh:
            for line in fh:
                line = line.strip()
                if not line:
                    continue
                event = json.loads(line)
                if event.get("kind") != "stage_compute_start":
                    continue
                payload = event.get("payload", {})
                if payload.get("phase") != "decode" or payload.get("stage") != 0:
                    continue
                capacity = payload.get("capacity_tokens", 0)
                res = payload.get("next_residual_tokens", 0)
                pre = payload.get("next_prefetched_tokens", 0)
                rows.append((payload.get("iter"), payload.get("exec_seconds"),
                             res / capacity if capacity else 0.0, pre / capacity if capacity else 0.0))
    except FileNotFoundError as exc:
        raise ConfigError(f"trace not found: {args.trace}") from exc
    except json.JSONDecodeError as exc:
        raise ConfigError(f"trace is not valid JSONL: {exc}") from exc
    with open(args.out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["iter", "exec_seconds", "resident_fraction", "prefetched_fraction"])
        for r in rows:
            w.writerow([r[0], f"{r[1]:.9f}", f"{r[2]:.6f}", f"{r[3]:.6f}"])
    print(f"wrote {len(rows)} iterations to {args.out}")
    return 0


def _workload_args(p):
    p.add_argument("--model", default="tiny-llama")
    p.add_argument("--requests", type=int, default=32)
    p.add_argument("--prompt", type=int, default=128)
    p.add_argument("--gen", type=int, default=32)
    p.add_argument("--micro-batches", type=int, default=4)
    p.add_argument("--pool-frac", type=float, default=0.75, help="KV pool cap as a fraction of peak KV")
    p.add_argument("--resident-frac", type=float, default=0.75, help="requests starting in HBM")
    p.add_argument("--pp", type=int, default=1, help="pipeline stages (single process)")
    p.add_argument("--seed", type=int, default=0)


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2605_02189_b200.cli", description=__doc__.splitlines()[0])
    sub = parser.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("decode", help="run the decode engine on a synthetic workload")
    _workload_args(p)
    p.add_argument("--horizon", type=int, default=None)
    p.add_argument("--prefill", action="store_true", help="seed KV with the real prefill instead of random KV")
    p.add_argument("--trace", default="trace.jsonl")
    p.add_argument("--metrics", default="metrics.json")
    p.set_defaults(fn=cmd_decode)
    p = sub.add_parser("prefill", help="prefill with layer-wise KV offload")
    _workload_args(p)
    p.add_argument("--staging", type=int, default=2, help="staging_pool_requests")
    p.add_argument("--trace", default="prefill_trace.jsonl")
    p.set_defaults(fn=cmd_prefill)
    p = sub.add_parser("calibrate", help="fit the decode-time estimator on this GPU")
    _workload_args(p)
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--samples", default="samples.csv")
    p.add_argument("--out", default="estimator.json")
    p.set_defaults(fn=cmd_calibrate)
    for name, fn, hlp in (("episode", cmd_episode, "prefill <-> decode episode (run_episode) on the GPU"),
                          ("compare", cmd_compare, "the same workload under several policies")):
        p = sub.add_parser(name, help=hlp)
        _workload_args(p)
        p.add_argument("--host-tokens", type=int, default=0, help="host KV capacity in tokens (0: unbounded)")
        p.add_argument("--rho-hi", type=float, default=0.9)
        p.add_argument("--horizon", type=int, default=None)
        if name == "episode":
            p.add_argument("--policy", default="dynamic")
            p.add_argument("--metrics", default="episode.json")
        else:
            p.add_argument("--policies", default="dynamic,no_prefetch,static:0.5")
            p.add_argument("--out", default="compare.csv")
        p.set_defaults(fn=fn)
    p = sub.add_parser("report", help="per-iteration decode series from a trace")
    p.add_argument("--trace", required=True)
    p.add_argument("--out", default="report.csv")
    p.set_defaults(fn=cmd_report)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    from .trace import CapacityError, OutOfMemory
    from .trace import ConfigError as TraceConfigError
    from .model_core import NoKvHeadroom
    try:
        return args.fn(args)
    except (ConfigError, TraceConfigError) as exc:
        print(f"config error: {exc}", file=sys.stderr)
        return 2
    except (CapacityError, OutOfMemory, NoKvHeadroom) as exc:
        print(f"runtime error: {exc}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
