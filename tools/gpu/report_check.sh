set -x
timeout 900 python -m pytest tests/test_report.py tests/test_groups.py tests/test_gpu_leveled.py tests/test_cpp_dropin.py -x -q 2>&1 | tail -15
