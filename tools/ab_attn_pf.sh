# A/B: per-warp L2 tensor prefetch of the KV blocks PM_ATTN_PF ahead of the attention ring
# (x the 2-D / 5-D pool map), single-lane stage shapes first, then C2.
OUT=${OUT:-gpurun_out/abpf}; mkdir -p $OUT
PM_ATTN_PF=4 timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q -k "paged_attention" > $OUT/t_pf4.log 2>&1; tail -1 $OUT/t_pf4.log
PM_ATTN_PF=4 timeout 600 python -m pytest tests/test_engine_gpu.py -x -q > $OUT/t_eng_pf4.log 2>&1; tail -1 $OUT/t_eng_pf4.log
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 6 --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for c in c3-stage c4-stage; do
  b ${c}_pf0 $c
  b ${c}_pf2 $c PM_ATTN_PF=2
  b ${c}_pf4 $c PM_ATTN_PF=4
  b ${c}_pf8 $c PM_ATTN_PF=8
  b ${c}_kv5pf4 $c PM_ATTN_PF=4 PM_ATTN_KV5=1
  b ${c}_kv5pf8 $c PM_ATTN_PF=8 PM_ATTN_KV5=1
done
b c2_pf0 c2; b c2_pf4 c2 PM_ATTN_PF=4; b c2_kv5pf4 c2 PM_ATTN_PF=4 PM_ATTN_KV5=1; b c2_pf0b c2; b c2_pf4b c2 PM_ATTN_PF=4
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ.get('OUT','gpurun_out/abpf')+'/*.json')):
    try:
        d=json.load(open(f)); a=d['roofline']['per_kind']['attention']
        print(os.path.basename(f), round(d['ms_per_step'],4), round(d['decode_roofline']['frac'],4), 'attn us', round(a['us_per_launch_exclusive'],2), 'GBps', round(a.get('GBps',0)), d['clocks']['sm_mhz'])
    except Exception as e: print(f, 'ERR', e)
PY
