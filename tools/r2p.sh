OUT=gpurun_out/r2p; mkdir -p $OUT
python tools/determinism.py 2>&1 | tail -1
PM_LANES=1 python tools/determinism.py 2>&1 | tail -1
PM_PDL=0 python tools/determinism.py 2>&1 | tail -1
PM_LANES=1 PM_PDL=0 python tools/determinism.py 2>&1 | tail -1
