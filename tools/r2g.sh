OUT=gpurun_out/r2g; mkdir -p $OUT
T=tests/test_pipeline_gpu.py
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest $T -x -q > $OUT/pipe_$i.log 2>&1; echo "run $i: $(tail -1 $OUT/pipe_$i.log)"; done
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
b c2_gather c2
b c3_gather c3-stage
timeout 300 python -m pytest tests/test_engine_gpu.py tests/test_seam_gpu.py -x -q > $OUT/pytest_kv.log 2>&1; tail -1 $OUT/pytest_kv.log
