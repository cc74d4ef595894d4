set -x
timeout 600 python -m pytest tests/test_gpu_packed.py -x -q 2>&1 | tail -30
timeout 900 python bench.py --steps 8 --warmup 3 --no-sort --c5-copies 0 --c4-layers 0 --leveled-models 0 --ingest-models 0 --no-cpu-baseline > gpurun_out/b_c3p.json 2> gpurun_out/b_c3p.err
python -c "
import json;d=json.load(open('gpurun_out/b_c3p.json'))['c3'];print(json.dumps(d['e2e']));print(json.dumps(d['e2e_dense']))"
tail -3 gpurun_out/b_c3p.err
