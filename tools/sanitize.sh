#!/bin/bash
# compute-sanitizer passes (memcheck, racecheck, synccheck, initcheck) over
# smoke() and the tiny engine parity test; logs under gpurun_out/sanitize_*.
# Usage (GPU box): bash tools/sanitize.sh
set -u
cd "$(dirname "$0")/.."
out=gpurun_out
mkdir -p $out
SMOKE='import __graft_entry__ as g; g.smoke()'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
      python -c "$SMOKE" > $out/sanitize_smoke_$tool.log 2>&1
  echo "smoke $tool rc=$?" >> $out/sanitize_summary.txt
done
for tool in memcheck racecheck synccheck; do
  PM_SANITIZE=1 timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
      python -m pytest -x -q -p no:cacheprovider "tests/test_engine_gpu.py::test_engine_matches_oracle_with_offload[2-False]" \
      > $out/sanitize_engine_$tool.log 2>&1
  echo "engine $tool rc=$?" >> $out/sanitize_summary.txt
done
