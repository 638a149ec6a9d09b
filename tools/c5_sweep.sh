#!/bin/bash
# BASELINE configs[4] (C5): PP=4 Qwen3-32B, sweep of batch size x micro-batch
# count, one stage (the last: 16 layers + lm_head) per run, offload on.
# Lines -> gpurun_out/c5/<config>.json; table: python tools/c5_table.py
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/c5
STEPS=${STEPS:-30}
for bs in 64 128 256 512 1024; do
  for m in 4 8 16; do
    c=c5-bs$bs-m$m
    timeout 600 python bench.py --config $c --steps $STEPS --warmup 5 --no-kernel-timing --no-cpu-baseline \
        --no-calibrate > gpurun_out/c5/$c.log 2>&1
    grep '^{' gpurun_out/c5/$c.log | tail -1 > gpurun_out/c5/$c.json
  done
done
