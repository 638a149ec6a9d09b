OUT=gpurun_out/r2i; mkdir -p $OUT
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_forward_ops_gpu.py tests/test_engine_gpu.py -x -q > $OUT/pytest_attn.log 2>&1; tail -3 $OUT/pytest_attn.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
timeout 120 python tools/attn_trace.py 768 qwen3-8b 36 121 > $OUT/trace_c2.txt 2>&1
timeout 120 python tools/attn_trace.py 1060 qwen3-32b 8 48 > $OUT/trace_c3.txt 2>&1
timeout 120 python tools/attn_trace.py 1060 llama3-70b 10 24 > $OUT/trace_c4.txt 2>&1
timeout 600 python tools/attn_sweep.py $OUT/attn_sweep.txt > $OUT/attn_sweep.log 2>&1
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for c in 1 2; do b c2_cfg$c c2 PM_ATTN_CFG=$c; b c3_cfg$c c3-stage PM_ATTN_CFG=$c; b c4_cfg$c c4-stage PM_ATTN_CFG=$c; done
