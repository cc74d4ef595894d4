# same-box A/B on C4 (28.6 M layers): lib/libxsp_v0.so (before) vs lib/libxsp.so, 2 alternations + parity
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_analysis_paths.py tests/test_timeshard.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
for i in 1 2; do
for L in libxsp_v0.so libxsp.so; do
  echo "== $L"; XSP_LIB=$PWD/paper_1908_06869_b200/lib/$L timeout 600 python tools/c4_stages.py 28600000 0.001 2>&1 | grep '"ms_wall"\|"names"\|"layers"\|"join"\|"fuse"'
done
done
