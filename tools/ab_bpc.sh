# attention KV blocks per work item in the real bench (PM_ATTN_BPC), launch config by the cost model
OUT=${OUT:-gpurun_out/abbpc}; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for bpc in 12 16 20 24 32; do b c3_$bpc c3-stage PM_ATTN_BPC=$bpc; done
for bpc in 12 16 24; do b c3cfg1_$bpc c3-stage PM_ATTN_BPC=$bpc PM_ATTN_CFG=1; done
for bpc in 12 16 20 24; do b c4_$bpc c4-stage PM_ATTN_BPC=$bpc; done
for bpc in 12 16 24; do b c2_$bpc c2 PM_ATTN_BPC=$bpc; done
