# quick C3 timing (3 runs) + parity smoke + pass1 launch list with DRAM bytes
set -x
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 3 --no-sort --c5-copies 0 --c4-layers 0 --leveled-models 0 --no-cpu-baseline"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
for i in 1 2 3; do timeout 300 $B | python tools/c3line.py; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_pass1 -c 4 --csv --log-file gpurun_out/launches_p1.csv $B --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_p1.csv
