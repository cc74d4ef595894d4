# full GPU test suite + default bench + reference arm
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
print('C5', round(d['value']), d['ms_per_step'], 'pipe', round(d['pipeline_roofline']['frac'],3), 'p1', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']), d['clocks'])
print('C3', round(d['c3']['value']), round(d['c3']['ms_per_step'],3), round(d['c3']['pipeline_roofline']['frac'],3))
print('C4', json.dumps(d.get('c4'))[:900])
print('LEV', json.dumps(d.get('leveled'))[:400])
print('ING', json.dumps(d.get('ingest_jsonl')))
print('SORT', json.dumps(d.get('sort_shuffled'))[:300])
print('CPU', json.dumps(d.get('cpu_baseline')))
PY
cat gpurun_out/bench_ref.json
