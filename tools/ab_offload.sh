# A/B of the decode offload path and the host replica placement (C2 bench line, short)
OUT=${OUT:-gpurun_out/ab}; mkdir -p $OUT
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
run kernel_numa PM_OFFLOAD_MODE=kernel
run dma_numa PM_OFFLOAD_MODE=dma
run dma_nonuma PM_OFFLOAD_MODE=dma PM_HOST_NUMA=-1
run kernel_nonuma PM_OFFLOAD_MODE=kernel PM_HOST_NUMA=-1

PM_OFFLOAD_MODE=dma timeout 300 python bench.py --config c3-stage --steps 40 --warmup 5 --no-kernel-timing --no-cpu-baseline > $OUT/c3_dma.json 2> $OUT/c3_dma.err
PM_OFFLOAD_MODE=dma PM_HOST_NUMA=-1 timeout 300 python bench.py --config c3-stage --steps 40 --warmup 5 --no-kernel-timing --no-cpu-baseline > $OUT/c3_dma_nonuma.json 2> $OUT/c3_dma_nonuma.err
