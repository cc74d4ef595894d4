set -x
timeout 900 python tools/e2e_packed_probe.py 12000000 2>&1 | tail -30
