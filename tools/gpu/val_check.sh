set -x
timeout 900 python -m pytest tests/test_gpu_validate.py tests/test_ingest.py tests/test_cpp_dropin.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 8 --warmup 3 --c5-copies 0 --c4-layers 0 --leveled-models 0 --ingest-models 0 --no-cpu-baseline > gpurun_out/bv.json 2> gpurun_out/bv.err
python -c "
import json;d=json.load(open('gpurun_out/bv.json'));print(json.dumps(d['validate']))" ; tail -2 gpurun_out/bv.err
timeout 600 python tools/ingest_probe.py 24 2>&1 | tail -14
