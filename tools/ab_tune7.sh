OUT=${OUT:-gpurun_out/abtune7}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_pipeline_gpu.py -x -q > $OUT/t.log 2>&1; tail -1 $OUT/t.log
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for r in a b; do b c2_$r c2; b c3_$r c3-stage; done
b c4 c4-stage; b c4_148 c4-stage PM_ATTN_SMS=148; b c3l c3-last
