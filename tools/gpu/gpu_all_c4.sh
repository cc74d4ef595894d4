set -x
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
L=$PWD/paper_1908_06869_b200/lib
for v in libxsp_base.so libxsp.so; do echo "== $v"; XSP_LIB=$L/$v timeout 600 python tools/c4_stages.py 28600000 0.001 2>&1 | tail -18 | tr -d '\n '; echo; done
