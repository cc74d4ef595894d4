# C4 stage split A/B: lib/libxsp_base.so (before) vs lib/libxsp.so, plus the analysis / correlate GPU tests and the full-size C4 diff
set -x
L=$PWD/paper_1908_06869_b200/lib
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_analysis_paths.py tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py tests/test_timeshard.py -x -q 2>&1 | tail -3
for v in libxsp_base.so libxsp.so; do echo "== $v"; XSP_LIB=$L/$v timeout 600 python tools/c4_stages.py 28600000 0.001 2>&1 | tail -18 | tr -d '\n '; echo; done
# XSP_FULLSCALE=1 timeout 1500 python -m pytest tests/test_gpu_fullsize.py -k c4_bench_size -x -q 2>&1 | tail -3
