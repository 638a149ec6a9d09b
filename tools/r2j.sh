OUT=gpurun_out/r2j; mkdir -p $OUT
timeout 900 python -m pytest tests/test_fused_fixup_gpu.py tests/test_kernels_gpu.py tests/test_post_variants_gpu.py -x -q > $OUT/pytest_fix.log 2>&1; tail -3 $OUT/pytest_fix.log
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
b c2_poll c2
b c2_post c2 PM_FIX_POLL=0
b c3_poll c3-stage
b c3_post c3-stage PM_FIX_POLL=0
b c4_poll c4-stage
b c4_post c4-stage PM_FIX_POLL=0
b c2_poll_b c2
