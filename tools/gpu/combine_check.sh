set -x
timeout 900 python -m pytest tests/test_shard.py tests/test_abi.py -x -q 2>&1 | tail -8
timeout 900 python bench.py --steps 4 --warmup 3 --c5-copies 0 --no-sort --no-cpu-baseline > gpurun_out/b_c3.json 2>gpurun_out/b_c3.err; tail -2 gpurun_out/b_c3.err
timeout 1200 python -c "
import sys, json; sys.argv=['bench.py','--steps','4','--warmup','3','--c5-copies','1','--no-sort','--no-cpu-baseline','--leveled-models','0','--e2e-steps','1']
import bench; bench.main()" > gpurun_out/b_c4.json 2>gpurun_out/b_c4.err; tail -3 gpurun_out/b_c4.err
python -c "import json;d=json.load(open('gpurun_out/b_c4.json'));print(json.dumps(d['c4']))"
