OUT=${OUT:-gpurun_out/abnonorm}; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star --no-calibrate > $OUT/$name.json 2> $OUT/$name.err; }
b c3 c3-stage; b c3_nonorm c3-stage PM_GEMM_DEBUG=256; b c4 c4-stage; b c4_nonorm c4-stage PM_GEMM_DEBUG=256
