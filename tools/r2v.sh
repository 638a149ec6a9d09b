timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -c "
import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import test_engine_gpu as t
t.test_engine_matches_oracle_with_offload(2, False)
print('engine test ok')
" > /tmp/rc2.log 2>&1; echo "rc=$?"; grep -v "^=========     " /tmp/rc2.log | tail -40
