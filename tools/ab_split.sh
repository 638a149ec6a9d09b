# two lanes on disjoint SM halves: GEMM workers / attention CTAs per lane
OUT=${OUT:-gpurun_out/absplit}; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
b c2_base c2
b c2_g74 c2 PM_GEMM_CTAS=74
b c2_g74_a74 c2 PM_GEMM_CTAS=74 PM_ATTN_SMS=74
b c2_g96 c2 PM_GEMM_CTAS=96
b c2_g96_a74 c2 PM_GEMM_CTAS=96 PM_ATTN_SMS=74
b c2_g148 c2 PM_GEMM_CTAS=148
b c2_a74 c2 PM_ATTN_SMS=74
b c2_base_b c2
