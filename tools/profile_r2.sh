# Round-2 measurement pass: GPU tests, bench lines (default / reference /
# per-stage), ncu launch list with DRAM traffic, full captures of the top kernels.
set -x
OUT=${OUT:-gpurun_out/r2a}; mkdir -p $OUT
nvidia-smi > $OUT/nvidia_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1
timeout 400 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 400 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/ref.err
for c in c3-last c3-stage c4-last c4-stage; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file $OUT/launches_traffic.csv python bench.py --steps 2 --warmup 3 --no-kernel-timing --no-cpu-baseline --no-calibrate --no-north-star > $OUT/ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:gemm_stream -s 400 -c 2 -o $OUT/gemm_full python bench.py --steps 2 --warmup 3 --no-kernel-timing --no-cpu-baseline --no-calibrate --no-north-star > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:paged_attn -s 100 -c 1 -o $OUT/attn_full python bench.py --steps 2 --warmup 3 --no-kernel-timing --no-cpu-baseline --no-calibrate --no-north-star > /dev/null 2>&1
ls -la $OUT
