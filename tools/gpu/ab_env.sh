# same-box A/B of one env switch ($AB_ENV, e.g. XSP_P1_REDUCE=tma = the "before"), C3 only, 3 alternations
set -x
B="python bench.py --steps 20 --warmup 3 --no-sort --c5-copies 0 --c4-layers 0 --leveled-models 0 --ingest-models 0 --no-cpu-baseline"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_packed.py tests/test_timeshard.py -x -q 2>&1 | tail -3
for i in 1 2 3; do
  env $AB_ENV timeout 300 $B | python tools/c3line.py
  timeout 300 $B | python tools/c3line.py
done
