OUT=gpurun_out/r2e; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
tail -3 $OUT/pytest_gpu.log
STEPS=30 bash tools/c5_sweep.sh
python tools/c5_table.py gpurun_out/c5 > $OUT/c5_table.md 2>&1
cat $OUT/c5_table.md
