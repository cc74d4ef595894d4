set -x
timeout 900 python -m pytest tests/test_ingest.py -x -q 2>&1 | tail -2
timeout 600 python tools/ingest_probe.py 24 2>&1 | tail -11
timeout 900 python bench.py --steps 4 --warmup 3 --c5-copies 1 --no-sort --c4-layers 0 --leveled-models 0 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bi.json 2> gpurun_out/bi.err
python tools/show.py gpurun_out/bi.json ingest_jsonl
tail -2 gpurun_out/bi.err
