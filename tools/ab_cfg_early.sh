# A/B after the early KV loads: attention warps x stages at C2 (default 12x2) and the C3 stage (default 8x3)
OUT=${OUT:-gpurun_out/abcfg}; mkdir -p $OUT
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 60 --warmup 6 --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for r in a b c; do b c2_def_$r c2; b c2_cfg2_$r c2 PM_ATTN_CFG=2; done
for r in a b; do b c3_def_$r c3-stage; b c3_cfg1_$r c3-stage PM_ATTN_CFG=1; b c3_cfg0_$r c3-stage PM_ATTN_CFG=0; done
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ.get('OUT','gpurun_out/abcfg')+'/*.json')):
    try:
        d=json.load(open(f)); a=d['roofline']['per_kind']['attention']
        print(os.path.basename(f), round(d['ms_per_step'],4), round(d['decode_roofline']['frac'],4), 'attn us', round(a['us_per_launch_exclusive'],2), 'GBps', round(a.get('GBps',0)), d['clocks']['sm_mhz'])
    except Exception as e: print(f, 'ERR', e)
PY
