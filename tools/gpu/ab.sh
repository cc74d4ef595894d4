B="python bench.py --steps 20 --warmup 3 --no-sort --c5 0 --c4-layers 0 --no-cpu-baseline"
for i in 1 2 3; do
for v in "" 1; do XSP_AB=$v timeout 300 $B | python -c "import json,sys;d=json.loads(sys.stdin.read());print('AB=$v',round(d['value']),round(d['ms_per_step'],4),{k:round(v,4) for k,v in d['stages_ms'].items()})"; done; done
