python tools/determinism_pipe.py 2>&1 | tail -1
PM_PDL=0 python tools/determinism_pipe.py 2>&1 | tail -1
for i in 1 2 3 4 5; do timeout 300 python -m pytest tests/test_pipeline_gpu.py -x -q > /tmp/p_$i.log 2>&1; echo "pipeline run $i: $(tail -1 /tmp/p_$i.log)"; done
for i in 1 2; do PM_FIX_POLL=1 timeout 300 python -m pytest tests/test_engine_gpu.py tests/test_pipeline_gpu.py tests/test_fused_fixup_gpu.py -x -q > /tmp/q_$i.log 2>&1; echo "poll tests $i: $(tail -1 /tmp/q_$i.log)"; grep FAILED /tmp/q_$i.log | head -3; done
