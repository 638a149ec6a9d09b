# A/B: C2 with / without the warm-up delta refit (same box, interleaved, default 60 steps)
OUT=${OUT:-gpurun_out/abrefit}; mkdir -p $OUT
b() { name=$1; shift; timeout 300 python bench.py "$@" --no-kernel-timing --no-cpu-baseline --no-north-star > $OUT/$name.json 2> $OUT/$name.err; }
for r in a b c; do b c2_refit_$r; b c2_norefit_$r --no-refit; done
b c3_refit --config c3-stage; b c3_norefit --config c3-stage --no-refit
python - <<'PY'
import json,glob,os
for f in sorted(glob.glob(os.environ.get('OUT','gpurun_out/abrefit')+'/*.json')):
    try:
        d=json.load(open(f)); k=d['kv_transfer']
        print(os.path.basename(f), round(d['ms_per_step'],4), round(d['decode_roofline']['frac'],4), d['rows_per_step'], d['estimator'].get('online_refit'), d['estimator']['step_fidelity'], 'd2h GB/s', round(k['d2h_GBps'],1), 'stall ms', round(k['exposed_stall_s']*1e3,2), d['clocks']['sm_mhz'])
    except Exception as e: print(f, 'ERR', e)
PY
