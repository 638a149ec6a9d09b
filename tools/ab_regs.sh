# Register caps so the other lane's small fixup CTAs can share SMs with attention / GEMM CTAs
OUT=${OUT:-gpurun_out/abregs}; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
b c2_base c2
b c2_attn128 c2 PM_B200_LIB=$PWD/gpurun_ab_attn128.so
b c2_rc128 c2 PM_B200_LIB=$PWD/gpurun_ab_rc128.so
b c2_base_b c2
b c3_base c3-stage
b c3_attn128 c3-stage PM_B200_LIB=$PWD/gpurun_ab_attn128.so
b c3_rc128 c3-stage PM_B200_LIB=$PWD/gpurun_ab_rc128.so
