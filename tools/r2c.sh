OUT=${OUT:-gpurun_out/r2c}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_fused_fixup_gpu.py -x -q > $OUT/pytest_fused.log 2>&1
tail -3 $OUT/pytest_fused.log
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_pipeline_gpu.py -x -q > $OUT/pytest_more.log 2>&1
tail -3 $OUT/pytest_more.log
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 5 --no-kernel-timing --no-cpu-baseline > $OUT/$name.json 2> $OUT/$name.err; }
b c3_fused c3-stage
b c3_post c3-stage PM_FUSED_FIXUP=0
b c4_fused c4-stage
b c4_post c4-stage PM_FUSED_FIXUP=0
b c3last_fused c3-last
