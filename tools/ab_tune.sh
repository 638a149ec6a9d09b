# GEMM worker span and the O/down norm form on the per-stage configs (single lane) and C2
OUT=${OUT:-gpurun_out/abtune}; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for n in 108 116 124 132 140 148; do b c3_ctas$n c3-stage PM_GEMM_CTAS_1LANE=$n; done
b c3_fusednorm c3-stage PM_SPLIT_NORM=0
for n in 108 116 132 148; do b c4_ctas$n c4-stage PM_GEMM_CTAS_1LANE=$n; done
b c4_fusednorm c4-stage PM_SPLIT_NORM=0
for n in 120 128 136; do b c2_ctas$n c2 PM_GEMM_CTAS=$n; done
b c2_splitnorm c2 PM_SPLIT_NORM=1
