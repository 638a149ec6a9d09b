# L2 run-ahead of each GEMM worker's next weight bytes while it waits on its input (env A/B)
OUT=${OUT:-gpurun_out/abahead}; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
b c3_0 c3-stage
b c3_128 c3-stage PM_PF_AHEAD_KB=128
b c3_256 c3-stage PM_PF_AHEAD_KB=256
b c3_512 c3-stage PM_PF_AHEAD_KB=512
b c3_0b c3-stage
b c4_0 c4-stage
b c4_256 c4-stage PM_PF_AHEAD_KB=256
b c2_0 c2
b c2_256 c2 PM_PF_AHEAD_KB=256
