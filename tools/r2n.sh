OUT=gpurun_out/r2n; mkdir -p $OUT
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_forward_ops_gpu.py tests/test_engine_gpu.py tests/test_fused_fixup_gpu.py -x -q > $OUT/pytest.log 2>&1; echo "tests: $(tail -1 $OUT/pytest.log)"
PM_FIX_POLL=1 timeout 300 python -m pytest tests/test_engine_gpu.py -x -q > $OUT/engine_poll.log 2>&1; echo "engine poll: $(tail -1 $OUT/engine_poll.log)"
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 120 python tools/attn_trace.py 768 qwen3-8b 36 121 > $OUT/trace_c2.txt 2>&1
timeout 120 python tools/attn_trace.py 1060 qwen3-32b 8 48 > $OUT/trace_c3.txt 2>&1
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for pm in 0 150 250; do b c2_pool$pm c2 PM_ATTN_POOL_PM=$pm; b c3_pool$pm c3-stage PM_ATTN_POOL_PM=$pm; b c4_pool$pm c4-stage PM_ATTN_POOL_PM=$pm; done
b c3_poll c3-stage PM_FIX_POLL=1
b c4_poll c4-stage PM_FIX_POLL=1
b c2_poll c2 PM_FIX_POLL=1
