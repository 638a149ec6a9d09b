# A/B: attention grid span (PM_ATTN_SMS) and warps x stages (PM_ATTN_CFG) at the C4 stage shape (24 rows)
OUT=${OUT:-gpurun_out/absms}; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 40 --warmup 6 --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for r in a b; do
  b c4_120_$r c4-stage; b c4_148_$r c4-stage PM_ATTN_SMS=148; b c4_136_$r c4-stage PM_ATTN_SMS=136
done
b c4_148_cfg1 c4-stage PM_ATTN_SMS=148 PM_ATTN_CFG=1; b c4_120_cfg1 c4-stage PM_ATTN_CFG=1
b c3_148 c3-stage PM_ATTN_SMS=148; b c3_120 c3-stage
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ.get('OUT','gpurun_out/absms')+'/*.json')):
    try:
        d=json.load(open(f)); a=d['roofline']['per_kind']['attention']
        print(os.path.basename(f), round(d['ms_per_step'],4), round(d['decode_roofline']['frac'],4), 'attn us', round(a['us_per_launch_exclusive'],2), 'GBps', round(a.get('GBps',0)), d['clocks']['sm_mhz'])
    except Exception as e: print(f, 'ERR', e)
PY
