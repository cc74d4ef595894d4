set -x
timeout 900 python -m pytest tests/test_gpu_leveled.py tests/test_gpu_packed.py -x -q 2>&1 | tail -4
timeout 900 python bench.py --steps 8 --warmup 3 --c5-copies 1 --no-sort --c4-layers 0 --ingest-models 0 --e2e-steps 1 --no-cpu-baseline > gpurun_out/lev.json 2> gpurun_out/lev.err
tail -2 gpurun_out/lev.err
python -c "
import json; d=json.load(open('gpurun_out/lev.json'))['leveled']
print({k: d[k] for k in ('value','ms_per_step','per_group_ms','stages_ms','roofline')})"
