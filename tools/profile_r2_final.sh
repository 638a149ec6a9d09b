# Round-2 final measurement pass (default build): GPU tests, smoke, bench lines
# (C2 default + reference arm + per-stage north-star configs), ncu launch lists
# with DRAM traffic (C2, C3 stage), full captures of the top kernels, the C5 sweep.
set -x
OUT=${OUT:-gpurun_out/r2final2}; mkdir -p $OUT
nvidia-smi > $OUT/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 400 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 400 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/ref.err
for c in c3-last c3-stage c4-last c4-stage; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file $OUT/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-kernel-timing --no-cpu-baseline --no-calibrate --no-north-star > $OUT/ncu_c2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file $OUT/launches_c3.csv python bench.py --config c3-stage --steps 2 --warmup 3 --no-kernel-timing --no-cpu-baseline --no-calibrate > $OUT/ncu_c3.log 2>&1
timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:gemm_stream -s 400 -c 2 -o $OUT/gemm_full python bench.py --steps 2 --warmup 3 --no-kernel-timing --no-cpu-baseline --no-calibrate --no-north-star > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:paged_attn -s 100 -c 1 -o $OUT/attn_full python bench.py --steps 2 --warmup 3 --no-kernel-timing --no-cpu-baseline --no-calibrate --no-north-star > /dev/null 2>&1
if [ -z "${SKIP_C5:-}" ]; then
  STEPS=30 bash tools/c5_sweep.sh
  python tools/c5_table.py gpurun_out/c5 > $OUT/c5_table.md 2>&1
fi
ls -la $OUT
