# round-2 status run: GPU tests, default bench, C3 whole-step launch list with DRAM bytes, ncu --set full of the top kernels
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-sort --c5-copies 0 --c4-layers 0"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_c3.csv $B > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pass1|k_p1_reduce|k_kernels|k_layers|k_names_fast|k_models" -s 8 -c 6 -o gpurun_out/c3_full $B > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -2; head -c 4000 gpurun_out/bench.json; cat gpurun_out/bench_ref.json
