OUT=gpurun_out/r2u; mkdir -p $OUT
for i in 1 2; do timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$i.log 2>&1; echo "suite $i: $(tail -1 $OUT/pytest_gpu_$i.log)"; grep FAILED $OUT/pytest_gpu_$i.log | head -3; done
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 30 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for r in a b; do b c2_flat_$r c2; b c2_stagger_$r c2 PM_LANE_PRIO=stagger; done
