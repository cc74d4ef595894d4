B="python bench.py --steps 10 --warmup 3 --no-sort --c5 0 --c4-layers 0 --no-cpu-baseline"
echo "== lanes (default)"; timeout 300 $B | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['stages_ms'])"
echo "== serial"; XSP_P1_SERIAL=1 XSP_P1_SERIAL_REDUCE=1 timeout 300 $B | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['stages_ms'])"
echo "== C4 2.86M cf=0.001"; timeout 600 python tools/c4_stages.py 2860000 0.001
echo "== C4 2.86M cf=0"; timeout 600 python tools/c4_stages.py 2860000 0
