OUT=gpurun_out/r2f; mkdir -p $OUT
T=tests/test_pipeline_gpu.py::test_pipeline_two_ranks_one_gpu_matches_single_process
for v in "PM_OFFLOAD_MODE=gather" "PM_OFFLOAD_MODE=dma" "PM_OFFLOAD_MODE=kernel" "PM_ATTN_BPC=12" "PM_OFFLOAD_MODE=gather"; do
  env $v timeout 300 python -m pytest $T -x -q > $OUT/pipe_${v}.log 2>&1; echo "$v: $(tail -1 $OUT/pipe_${v}.log)"
done
timeout 600 python -m pytest tests/test_engine_gpu.py tests/test_seam_gpu.py tests/test_prefill_gpu.py tests/test_episode_gpu.py -x -q > $OUT/pytest_kv.log 2>&1; tail -1 $OUT/pytest_kv.log
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 30 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
b c2_gather c2
b c2_dma c2 PM_OFFLOAD_MODE=dma
b c3_gather c3-stage
b c3_dma c3-stage PM_OFFLOAD_MODE=dma
