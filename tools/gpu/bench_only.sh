set -x
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
print('C5', round(d['value']), d['ms_per_step'], 'pipe', round(d['pipeline_roofline']['frac'],3), 'p1', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']), d['clocks'])
print('C3', round(d['c3']['value']), round(d['c3']['ms_per_step'],3), round(d['c3']['pipeline_roofline']['frac'],3), 'e2e', round(d['c3']['e2e']['value']), 'full', round(d['c3']['e2e_full']['value']), 'dense', round(d['c3']['e2e_dense']['value']))
for k in ('c4','leveled','ingest_jsonl','sort_shuffled','validate','cpu_baseline'):
    v = d.get(k) or {}
    print(k, {kk: v.get(kk) for kk in ('value','ms_per_step','per_group_ms','spans') if kk in v})
PY
