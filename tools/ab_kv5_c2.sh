# C2 repeats of the attention-map A/B (two lanes: noisier than the single-lane stages), plus the GPU suite.
OUT=${OUT:-gpurun_out/abkv5c2}; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; tail -1 $OUT/pytest_gpu.log
b() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 60 --warmup 6 --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for r in a b c; do b c2_kv5_$r c2; b c2_kv2_$r c2 PM_ATTN_KV5=0; done
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ.get('OUT','gpurun_out/abkv5c2')+'/*.json')):
    try:
        d=json.load(open(f))
        print(os.path.basename(f), round(d['ms_per_step'],4), round(d['decode_roofline']['frac'],4), round(d['rows_per_step'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])
    except Exception as e: print(f, 'ERR', e)
PY
