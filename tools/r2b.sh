OUT=gpurun_out/r2b; mkdir -p $OUT
timeout 600 python -m pytest tests/test_engine_gpu.py tests/test_seam_gpu.py -x -q > $OUT/pytest_kv.log 2>&1
timeout 300 python bench.py --steps 30 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/c2.json 2> $OUT/c2.err
for c in c3-stage c4-stage c3-last; do timeout 300 python bench.py --config $c --no-cpu-baseline > $OUT/$c.json 2> $OUT/$c.err; done
timeout 900 python tools/attn_sweep.py $OUT/attn_sweep.txt > $OUT/attn_sweep.log 2>&1
