# GPU tests + C4 stage breakdown + full default bench
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 900 python tools/c4_stages.py 28600000 0.001 > gpurun_out/c4_stages.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/c4_stages.log; python -c "
import json;d=json.load(open('gpurun_out/bench.json'))
print('C5', round(d['value']), d['ms_per_step'], d['pipeline_roofline']['frac'], d['roofline']['frac'], 'e2e', round(d['e2e']['value']))
print('C3', round(d['c3']['value']), d['c3']['ms_per_step'], d['c3']['pipeline_roofline']['frac'])
print('C4', json.dumps(d.get('c4')))
print('LEV', json.dumps(d.get('leveled')))
"; tail -5 gpurun_out/bench.err
