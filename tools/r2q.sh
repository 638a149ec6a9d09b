python tools/determinism_pipe.py 2>&1 | tail -1
PM_PDL=0 python tools/determinism_pipe.py 2>&1 | tail -1
PM_OFFLOAD_MODE=dma python tools/determinism_pipe.py 2>&1 | tail -1
