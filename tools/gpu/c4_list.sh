set -x
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4b.csv python tools/c4_stages.py 5000000 0.001 > gpurun_out/ncu_c4b.log 2>&1
python tools/launches.py gpurun_out/launches_c4b.csv | head -40
