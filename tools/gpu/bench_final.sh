# default bench + reference arm + smoke (round-end numbers)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -1 gpurun_out/smoke.log; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
print('C5', round(d['value']), d['ms_per_step'], 'pipe', round(d['pipeline_roofline']['frac'],3), 'p1', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']), d['clocks'])
print('C3', round(d['c3']['value']), round(d['c3']['ms_per_step'],3), 'e2e', round(d['c3']['e2e']['value']))
print('C4', round(d['c4']['value']), d['c4']['ms_per_step'])
r=json.load(open('gpurun_out/bench_ref.json')); print('REF', r['value'])
PY
