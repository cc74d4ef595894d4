# same-box A/B of k_pass1 (lib/libxsp_base.so = before, lib/libxsp.so = after) + packed-input tests + e2e C3
set -x
B="python bench.py --steps 20 --warmup 3 --no-sort --c5-copies 0 --c4-layers 0 --leveled-models 0 --ingest-models 0 --no-cpu-baseline"
timeout 600 python -m pytest tests/test_gpu_packed.py tests/test_gpu_parity.py -x -q 2>&1 | tail -4
for i in 1 2 3; do
  XSP_LIB=$PWD/paper_1908_06869_b200/lib/libxsp_base.so timeout 300 $B | python tools/c3line.py
  timeout 300 $B | python tools/c3line.py
done
