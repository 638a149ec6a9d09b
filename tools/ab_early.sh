# A/B: attention KV loads ahead of the PDL dependency wait (PM_ATTN_EARLY=1, default) vs after (0)
OUT=${OUT:-gpurun_out/abearly}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_pipeline_gpu.py tests/test_prefill_gpu.py -x -q > $OUT/t.log 2>&1; tail -1 $OUT/t.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; tail -1 $OUT/smoke.log
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 60 --warmup 6 --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for r in a b; do
  b c3_on_$r c3-stage; b c3_off_$r c3-stage PM_ATTN_EARLY=0
  b c4_on_$r c4-stage; b c4_off_$r c4-stage PM_ATTN_EARLY=0
  b c2_on_$r c2; b c2_off_$r c2 PM_ATTN_EARLY=0
done
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ.get('OUT','gpurun_out/abearly')+'/*.json')):
    try:
        d=json.load(open(f)); a=d['roofline']['per_kind']['attention']
        print(os.path.basename(f), round(d['ms_per_step'],4), round(d['decode_roofline']['frac'],4), 'attn us', round(a['us_per_launch_exclusive'],2), 'GBps', round(a.get('GBps',0)), d['clocks']['sm_mhz'])
    except Exception as e: print(f, 'ERR', e)
PY
