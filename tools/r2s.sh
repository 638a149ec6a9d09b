OUT=gpurun_out/r2s; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
PM_SANITIZE=1 timeout 2400 compute-sanitizer --tool racecheck --print-limit 50 --error-exitcode 9 python -m pytest -x -q -p no:cacheprovider "tests/test_engine_gpu.py::test_engine_matches_oracle_with_offload[2-False]" > $OUT/sanitize_engine_racecheck.log 2>&1; echo "engine racecheck rc=$?"
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 --error-exitcode 9 python -m pytest -x -q -p no:cacheprovider "tests/test_engine_gpu.py::test_engine_matches_oracle_with_offload[1-True]" > $OUT/sanitize_engine2lane_memcheck.log 2>&1; echo "engine 2-lane memcheck rc=$?"
