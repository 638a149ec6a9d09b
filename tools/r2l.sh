OUT=gpurun_out/r2l; mkdir -p $OUT
timeout 180 python -m pytest tests/test_engine_gpu.py -x -q > $OUT/engine.log 2>&1; echo "engine poll: $? $(tail -1 $OUT/engine.log)"
PM_FIX_POLL=0 timeout 180 python -m pytest tests/test_engine_gpu.py -x -q > $OUT/engine_post.log 2>&1; echo "engine post: $? $(tail -1 $OUT/engine_post.log)"
timeout 300 python bench.py --steps 20 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/c2.json 2> $OUT/c2.err; echo "c2 bench: $?"
