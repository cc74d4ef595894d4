set -x
timeout 900 python -m pytest tests/test_ingest.py tests/test_report.py tests/test_shard.py -x -q 2>&1 | tail -25
