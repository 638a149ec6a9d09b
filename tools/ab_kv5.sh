# A/B: attention KV blocks as one 5-D TMA copy (PM_ATTN_KV5=1, default) vs four 2-D boxes (0).
OUT=${OUT:-gpurun_out/abkv5}; mkdir -p $OUT
timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -x -q > $OUT/t_kv5.log 2>&1; tail -1 $OUT/t_kv5.log
PM_ATTN_KV5=0 timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k attn > $OUT/t_kv2.log 2>&1; tail -1 $OUT/t_kv2.log
for i in 1 2 3; do timeout 300 python -m pytest tests/test_pipeline_gpu.py -x -q > $OUT/t_pipe_$i.log 2>&1; tail -1 $OUT/t_pipe_$i.log; done
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 6 --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for r in a b; do
  b c3_kv5_$r c3-stage; b c3_kv2_$r c3-stage PM_ATTN_KV5=0
  b c4_kv5_$r c4-stage; b c4_kv2_$r c4-stage PM_ATTN_KV5=0
done
b c2_kv5 c2; b c2_kv2 c2 PM_ATTN_KV5=0
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ.get('OUT','gpurun_out/abkv5')+'/*.json')):
    try:
        d=json.load(open(f)); a=d['roofline']['per_kind']['attention']
        print(os.path.basename(f), round(d['ms_per_step'],4), round(d['decode_roofline']['frac'],4), 'attn us', round(a['us_per_launch_exclusive'],2), 'GBps', round(a.get('GBps',0)), d['clocks']['sm_mhz'])
    except Exception as e: print(f, 'ERR', e)
PY
