OUT=${OUT:-gpurun_out/abtune2}; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for r in a b; do for n in 128 136 144; do b c2_ctas${n}_$r c2 PM_GEMM_CTAS=$n; done; done
for r in a b; do b c3_split_$r c3-stage; b c3_fused_$r c3-stage PM_SPLIT_NORM=0; done
