# Quick verification pass of the current build: GPU tests, smoke, default bench line, reference arm.
set -x
OUT=${OUT:-gpurun_out/verify}; mkdir -p $OUT
nvidia-smi > $OUT/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke=$?
timeout 400 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo bench=$?
timeout 400 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/ref.err; echo ref=$?
