# C4 stage breakdown + launch list (time + DRAM bytes) of one correlate+analyze of a 5M-layer C4 trace;
# and the N=2 bench path (two ranks sharing the one GPU over gloo) with the time-sharded C4
set -x
mkdir -p gpurun_out
timeout 900 python tools/c4_stages.py 28600000 0.001 > gpurun_out/c4_stages.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python tools/c4_stages.py 5000000 0.001 > gpurun_out/ncu_c4.log 2>&1
XSP_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --c5-copies 2 --no-sort --c4-layers 2000000 --no-cpu-baseline > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
cat gpurun_out/c4_stages.log; tail -c 3000 gpurun_out/bench_n2.json; tail -20 gpurun_out/bench_n2.err
