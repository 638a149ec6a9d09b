OUT=${OUT:-gpurun_out/abtune4}; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for r in a b; do b c2_def_$r c2; b c2_attn8x3_$r c2 PM_ATTN_CFG=2; b c2_pair32_$r c2 PM_PAIR_MAX_UNITS=32; done
b c2_pair100 c2 PM_PAIR_MAX_UNITS=100
