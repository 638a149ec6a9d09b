OUT=gpurun_out/r2m; mkdir -p $OUT
T="tests/test_engine_gpu.py::test_engine_matches_oracle_with_offload"
timeout 180 python -m pytest "$T[2-False]" -x -q > $OUT/pp2.log 2>&1; echo "pp2 eager 1-lane poll: $(tail -1 $OUT/pp2.log)"
PM_LANES=1 timeout 180 python -m pytest "$T[1-True]" -x -q > $OUT/l1g.log 2>&1; echo "pp1 graphs 1-lane poll: $(tail -1 $OUT/l1g.log)"
PM_LANES=2 timeout 180 python -m pytest "$T[1-True]" -x -q > $OUT/l2g.log 2>&1; echo "pp1 graphs 2-lane poll: $(tail -1 $OUT/l2g.log)"
PM_LANES=2 PM_PDL=0 timeout 180 python -m pytest "$T[1-True]" -x -q > $OUT/l2g_nopdl.log 2>&1; echo "pp1 graphs 2-lane poll no-PDL: $(tail -1 $OUT/l2g_nopdl.log)"
