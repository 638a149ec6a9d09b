OUT=gpurun_out/r2y; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
b c2 c2; b c3 c3-stage; b c4 c4-stage; b c2b c2
timeout 300 python -m pytest tests/test_engine_gpu.py tests/test_offload_gpu.py tests/test_host_abi.py -x -q > $OUT/t.log 2>&1; tail -1 $OUT/t.log
