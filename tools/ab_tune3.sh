OUT=${OUT:-gpurun_out/abtune3}; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for n in 132 136 140; do b c2_ctas${n} c2 PM_GEMM_CTAS=$n; done
b c2_ctas136_c c2 PM_GEMM_CTAS=136
for r in a b; do b c4_split_$r c4-stage; b c4_fused_$r c4-stage PM_SPLIT_NORM=0; done
b c3l_split c3-last; b c3l_fused c3-last PM_SPLIT_NORM=0
