# per-kernel launch list (time + DRAM bytes) of C3 bench steps, and one full ncu capture of the top kernels
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-sort --c5 0 --c4-layers 0"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_c3_${TAG}.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_pass1|k_p1_reduce|k_kernels|k_layers|k_names_fast|k_models" -s 8 -c 6 -o gpurun_out/c3_${TAG} $B > gpurun_out/ncu_full_${TAG}.log 2>&1
ls -la gpurun_out
