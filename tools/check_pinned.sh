# pinned-replica robustness: offload/engine/seam/prefill tests over the chunked replica, a full GPU suite, benches
OUT=${OUT:-gpurun_out/pinned}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_offload_gpu.py tests/test_engine_gpu.py tests/test_seam_gpu.py tests/test_prefill_gpu.py tests/test_episode_gpu.py -x -q > $OUT/t.log 2>&1; tail -1 $OUT/t.log; grep FAILED $OUT/t.log | head
timeout 1500 python -m pytest tests -m gpu -q > $OUT/suite.log 2>&1; tail -1 $OUT/suite.log; grep FAILED $OUT/suite.log | head
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 30 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
b c2 c2; b c3 c3-stage
