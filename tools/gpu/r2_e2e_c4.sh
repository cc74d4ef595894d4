# packed / rows-only tests, C3 e2e lines, C4 stage split, one ncu capture of the main C4 analysis kernels
set -x
timeout 900 python -m pytest tests/test_gpu_packed.py tests/test_gpu_parity.py tests/test_timeshard.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --steps 8 --warmup 3 --no-sort --c5-copies 0 --c4-layers 0 --leveled-models 0 --ingest-models 0 --no-cpu-baseline > gpurun_out/e2e.json 2> gpurun_out/e2e.err
python -c "
import json; d=json.load(open('gpurun_out/e2e.json'))['c3']
for k in ('e2e','e2e_full','e2e_dense'): print(k, round(d[k]['value']), round(d[k]['ms_per_step'],2), d[k]['h2d_bytes_per_step'], d[k]['d2h_bytes_per_step'])
print('c3', round(d['value']))"
timeout 900 python tools/c4_stages.py 28600000 0.001 2>&1 | tail -16
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'k_names_fast|k_layers|k_big_chunks|k_gather_kernels|k_fuse|k_join_insert|k_kernels_r1|k_pass1' -s 20 -c 8 \
  -o gpurun_out/ncu_c4_multi python tools/c4_stages.py 5000000 0.001 > gpurun_out/ncu_c4_multi.log 2>&1
tail -3 gpurun_out/ncu_c4_multi.log
