OUT=${OUT:-gpurun_out/abtune6}; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for n in 96 104 112 120 128; do b c2_attn$n c2 PM_ATTN_SMS=$n; done
b c2_attn112_g144 c2 PM_ATTN_SMS=112 PM_GEMM_CTAS=144
b c2_attn120_g128 c2 PM_ATTN_SMS=120 PM_GEMM_CTAS=128
b c3_attn120 c3-stage PM_ATTN_SMS=120
