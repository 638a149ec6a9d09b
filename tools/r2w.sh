timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -X faulthandler -c "
import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
print('start', flush=True)
import test_engine_gpu as t
t.test_engine_matches_oracle_with_offload(2, False)
print('engine test ok', flush=True)
" > /tmp/rc3.log 2>&1; echo "engine rc=$?"; grep -v "^=========     " /tmp/rc3.log | tail -25
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest -x -q -p no:cacheprovider tests/test_kernels_gpu.py -k "attention" > /tmp/rc4.log 2>&1; echo "attention kernels racecheck rc=$?"; tail -4 /tmp/rc4.log
