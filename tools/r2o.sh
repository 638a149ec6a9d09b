OUT=gpurun_out/r2o; mkdir -p $OUT
for i in 1 2 3 4 5 6 7 8; do timeout 300 python -m pytest tests/test_pipeline_gpu.py -x -q > $OUT/pipe_$i.log 2>&1; echo "pipeline run $i: $(tail -1 $OUT/pipe_$i.log)"; done
for i in 1 2 3; do PM_FIX_POLL=1 timeout 300 python -m pytest tests/test_engine_gpu.py tests/test_pipeline_gpu.py tests/test_fused_fixup_gpu.py -x -q > $OUT/poll_$i.log 2>&1; echo "poll tests $i: $(tail -1 $OUT/poll_$i.log)"; done
timeout 300 python -m pytest tests/test_calibrate_gpu.py -x -q > $OUT/calib.log 2>&1; echo "calibrate: $(tail -1 $OUT/calib.log)"
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 30 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for r in a b; do
  b c3_post_$r c3-stage; b c3_poll_$r c3-stage PM_FIX_POLL=1
  b c4_post_$r c4-stage; b c4_poll_$r c4-stage PM_FIX_POLL=1
  b c2_post_$r c2; b c2_poll_$r c2 PM_FIX_POLL=1
done
