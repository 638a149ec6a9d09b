OUT=${OUT:-gpurun_out/abtune5}; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for r in a b; do b c2_def_$r c2; b c2_attn136_$r c2 PM_ATTN_SMS=136; b c2_attn120_$r c2 PM_ATTN_SMS=120; done
b c3_def c3-stage; b c3_attn136 c3-stage PM_ATTN_SMS=136
