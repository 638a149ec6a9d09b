OUT=${OUT:-gpurun_out/vb}; mkdir -p $OUT
timeout 400 python bench.py > $OUT/bench.json 2> $OUT/bench.err
for c in c4-last c4-stage; do timeout 300 python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2> $OUT/bench_$c.err; done
python - <<'PY'
import json,os
o=os.environ.get('OUT','gpurun_out/vb')
for f in ['bench.json','bench_c4-last.json','bench_c4-stage.json']:
    d=json.load(open(f'{o}/{f}')); print(f, round(d['value']), round(d['ms_per_step'],3), round(d['decode_roofline']['frac'],3), d['estimator'].get('online_refit'), d['estimator']['step_fidelity'], d['clocks'])
    for st in d.get('north_star',{}).get('stages',[]): print('  ', st['config'], round(st['ms_per_step'],3), round(st['decode_roofline_frac'],3), st['estimator_fidelity'], st.get('online_refit'))
PY
