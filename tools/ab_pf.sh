# L2 prefetch of the next projection's first bytes (single-lane per-stage runs) + attention chunk sweep
OUT=${OUT:-gpurun_out/abpf}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q > $OUT/pytest_kernels.log 2>&1
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 5 --no-kernel-timing --no-cpu-baseline > $OUT/$name.json 2> $OUT/$name.err; }
b c3_pf0 c3-stage PM_PF_MB=0
b c3_pf8 c3-stage PM_PF_MB=8
b c3_pf16 c3-stage PM_PF_MB=16
b c3_pf32 c3-stage PM_PF_MB=32
b c3_pf16_contig c3-stage PM_PF_MB=16 PM_PF_STRIPES=0
b c3_pf16_qkv c3-stage PM_PF_MB=16 PM_PF_QKV=1
b c3_pf0_b c3-stage PM_PF_MB=0
b c4_pf0 c4-stage PM_PF_MB=0
b c4_pf16 c4-stage PM_PF_MB=16
b c4_pf32 c4-stage PM_PF_MB=32
timeout 900 python tools/attn_sweep.py $OUT/attn_sweep.txt > $OUT/attn_sweep.log 2>&1
