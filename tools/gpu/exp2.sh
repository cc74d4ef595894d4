timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
B="python bench.py --steps 10 --warmup 3 --no-sort --c5 0 --c4-layers 0 --no-cpu-baseline"
timeout 300 $B | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d['stages_ms'])"
timeout 900 python tools/c4_stages.py 28600000 0.001
