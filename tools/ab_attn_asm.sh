OUT=${OUT:-gpurun_out/abasm}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -x -q > $OUT/t.log 2>&1; tail -1 $OUT/t.log
timeout 120 python tools/attn_trace.py 768 qwen3-8b 36 121 > $OUT/trace_c2.txt 2>&1
PM_B200_LIB=$PWD/gpurun_ab_attnvol.so timeout 120 python tools/attn_trace.py 768 qwen3-8b 36 121 > $OUT/trace_c2_vol.txt 2>&1
timeout 120 python tools/attn_trace.py 1060 qwen3-32b 8 48 > $OUT/trace_c3.txt 2>&1
PM_B200_LIB=$PWD/gpurun_ab_attnvol.so timeout 120 python tools/attn_trace.py 1060 qwen3-32b 8 48 > $OUT/trace_c3_vol.txt 2>&1
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for r in a b; do b c2_pure_$r c2; b c2_vol_$r c2 PM_B200_LIB=$PWD/gpurun_ab_attnvol.so; b c3_pure_$r c3-stage; b c3_vol_$r c3-stage PM_B200_LIB=$PWD/gpurun_ab_attnvol.so; done
