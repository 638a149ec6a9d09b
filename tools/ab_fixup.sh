# Upper bound of removing the fixup/norm launches: PM_GEMM_DEBUG=16 skips them (wrong numerics, timing only)
OUT=${OUT:-gpurun_out/abfix}; mkdir -p $OUT
for c in c3-stage c4-stage; do
  timeout 300 python bench.py --config $c --steps 40 --warmup 5 --no-kernel-timing --no-cpu-baseline > $OUT/$c.json 2> $OUT/$c.err
  PM_GEMM_DEBUG=16 timeout 300 python bench.py --config $c --steps 40 --warmup 5 --no-kernel-timing --no-cpu-baseline > $OUT/${c}_nofix.json 2> $OUT/${c}_nofix.err
done
timeout 300 python bench.py --steps 30 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/c2.json 2> $OUT/c2.err
PM_GEMM_DEBUG=16 timeout 300 python bench.py --steps 30 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/c2_nofix.json 2> $OUT/c2_nofix.err
