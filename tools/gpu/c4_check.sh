set -x
timeout 900 python -m pytest tests/test_timeshard.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
timeout 900 python tools/c4_stages.py 28600000 0.001 2>&1 | tail -16
