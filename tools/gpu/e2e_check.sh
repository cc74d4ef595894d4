# packed-input tests + the C3 e2e lines (rows-only / full / dense)
set -x
timeout 900 python -m pytest tests/test_gpu_packed.py -x -q 2>&1 | tail -15
timeout 600 python bench.py --steps 8 --warmup 3 --no-sort --c5-copies 0 --c4-layers 0 --leveled-models 0 --ingest-models 0 --no-cpu-baseline > gpurun_out/e2e.json 2> gpurun_out/e2e.err
tail -3 gpurun_out/e2e.err
python tools/e2eline.py gpurun_out/e2e.json
