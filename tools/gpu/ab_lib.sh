# same-box A/B: lib/libxsp_base.so (before) vs lib/libxsp.so (after), C3 only, 3 alternations, + analysis tests
set -x
B="python bench.py --steps 20 --warmup 3 --no-sort --c5-copies 0 --c4-layers 0 --leveled-models 0 --ingest-models 0 --no-cpu-baseline"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_timeshard.py tests/test_gpu_pipeline.py tests/test_gpu_packed.py -x -q 2>&1 | tail -2
for i in 1 2 3; do
  XSP_LIB=$PWD/paper_1908_06869_b200/lib/libxsp_base.so timeout 300 $B | python tools/c3line.py
  timeout 300 $B | python tools/c3line.py
done
