OUT=gpurun_out/r2k; mkdir -p $OUT
timeout 180 python -m pytest tests/test_engine_gpu.py -x -q > $OUT/engine.log 2>&1; echo "engine tiny 2-lane: $? $(tail -1 $OUT/engine.log)"
cat > /tmp/lanes.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2605_02189_b200.engine import DecodeEngine
lanes = int(sys.argv[1])
spec, state, cfg, params, reqs, desc = bench.workload()
eng = DecodeEngine(spec, state, cfg, params, reqs, device="cuda:0", kv_init="random", timing=True, seed=0, calibrate=False, lanes=lanes)
for i in range(12):
    eng.step()
    torch.cuda.synchronize()
    print("step", i, flush=True)
print("ok", lanes)
PY
timeout 120 python /tmp/lanes.py 1 > $OUT/c2_lanes1.log 2>&1; echo "c2 lanes=1: $? $(tail -1 $OUT/c2_lanes1.log)"
timeout 120 python /tmp/lanes.py 2 > $OUT/c2_lanes2.log 2>&1; echo "c2 lanes=2: $? $(tail -1 $OUT/c2_lanes2.log)"
