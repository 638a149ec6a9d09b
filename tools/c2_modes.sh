# Repeated C2 lines with the in-process HBM copy probe and host placement (slow-mode hunt)
OUT=${OUT:-gpurun_out/c2modes}; mkdir -p $OUT
for i in 1 2 3 4 5 6 7; do
  timeout 300 python bench.py --no-cpu-baseline --no-north-star > $OUT/c2_$i.json 2> $OUT/c2_$i.err
done
python - <<'PY'
import json,glob,os
o=os.environ.get('OUT','gpurun_out/c2modes')
for i in range(1,8):
    try:
        d=json.load(open(f'{o}/c2_{i}.json')); r=d['decode_roofline']; pk=d['roofline']['per_kind']
        print(i, round(d['ms_per_step'],3), 'hbm', round(r['hbm_probe_GBps']), r['host'], 'gemm us', round(pk['gemm']['us_per_launch_exclusive'],2), 'attn us', round(pk['attention']['us_per_launch_exclusive'],2), 'd2h', round(d['kv_transfer']['d2h_GBps'],1), d['clocks']['sm_mhz'])
    except Exception as e: print(i, 'ERR', e)
PY
