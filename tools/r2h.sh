OUT=gpurun_out/r2h; mkdir -p $OUT
timeout 120 python tools/attn_trace.py 768 qwen3-8b 36 121 > $OUT/trace_c2.txt 2>&1
timeout 120 python tools/attn_trace.py 1060 qwen3-32b 8 48 > $OUT/trace_c3.txt 2>&1
timeout 120 python tools/attn_trace.py 1060 llama3-70b 10 24 > $OUT/trace_c4.txt 2>&1
EXTRA_DEBUG=1 timeout 120 python tools/attn_trace.py 768 qwen3-8b 36 121 > $OUT/trace_c2_memonly.txt 2>&1
EXTRA_DEBUG=1 timeout 120 python tools/attn_trace.py 1060 qwen3-32b 8 48 > $OUT/trace_c3_memonly.txt 2>&1
timeout 600 python -m pytest tests/test_offload_gpu.py -x -q > $OUT/pytest_offload.log 2>&1; tail -1 $OUT/pytest_offload.log
