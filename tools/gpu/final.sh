# full GPU suite + default bench + reference arm + C3 whole-step launch list (DRAM) + ncu --set full of the top kernels
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-sort --c5-copies 0 --c4-layers 0 --leveled-models 0 --ingest-models 0"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 140 --csv --log-file gpurun_out/launches_c3_r2f.csv $B > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pass1|k_p1_reduce|k_kernels|k_layers|k_names_fast|k_models|k_group_check" -s 8 -c 7 -o gpurun_out/c3_full_r2f $B > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
print('C5', round(d['value']), d['ms_per_step'], 'pipe', round(d['pipeline_roofline']['frac'],3), 'p1', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']), d['clocks'])
print('C3', round(d['c3']['value']), round(d['c3']['ms_per_step'],3), round(d['c3']['pipeline_roofline']['frac'],3), 'e2e', round(d['c3']['e2e']['value']), 'dense', round(d['c3']['e2e_dense']['value']))
for k in ('c4','leveled','ingest_jsonl','sort_shuffled','validate','cpu_baseline'):
    print(k, json.dumps(d.get(k))[:500])
PY
cat gpurun_out/bench_ref.json | head -c 600
