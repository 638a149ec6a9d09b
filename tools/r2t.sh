python tools/determinism_pp2.py 2>&1 | tail -1
PM_PDL=0 python tools/determinism_pp2.py 2>&1 | tail -1
PM_OFFLOAD_MODE=dma python tools/determinism_pp2.py 2>&1 | tail -1
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest -x -q -p no:cacheprovider "tests/test_engine_gpu.py::test_engine_matches_oracle_with_offload[2-False]" > /tmp/rc.log 2>&1; echo "racecheck rc=$?"; tail -30 /tmp/rc.log
