set -x
OUT=${OUT:-gpurun_out/r1g}; mkdir -p $OUT
timeout 400 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 400 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/ref.err
timeout 300 python bench.py --config c3-stage --no-cpu-baseline --no-calibrate > $OUT/bench_c3.json 2>/dev/null
timeout 300 python bench.py --config c4-stage --no-cpu-baseline --no-calibrate > $OUT/bench_c4.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv --log-file $OUT/launches_traffic.csv python bench.py --steps 2 --warmup 3 --no-kernel-timing --no-cpu-baseline --no-calibrate > $OUT/ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:gemm_stream -s 400 -c 2 -o $OUT/gemm_full python bench.py --steps 2 --warmup 3 --no-kernel-timing --no-cpu-baseline --no-calibrate > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:paged_attn -s 100 -c 1 -o $OUT/attn_full python bench.py --steps 2 --warmup 3 --no-kernel-timing --no-cpu-baseline --no-calibrate > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --cache-control none --clock-control none -k regex:gemm_reduce_v4 -s 10 -c 1 -o $OUT/post_full python bench.py --steps 2 --warmup 3 --no-kernel-timing --no-cpu-baseline --no-calibrate > /dev/null 2>&1
ls -la $OUT
