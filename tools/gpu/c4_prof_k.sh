# one ncu --set full capture of a C4 kernel (5 M layers): KERNEL=k_join_check bash tools/gpu/c4_prof_k.sh
set -x
K=${KERNEL:-k_join_check}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-1} -c 1 \
  -o gpurun_out/ncu_c4_$K python tools/c4_stages.py 5000000 0.001 > gpurun_out/ncu_c4_$K.log 2>&1
tail -3 gpurun_out/ncu_c4_$K.log
timeout 1200 python tools/c4_stages.py 28600000 0.001 2>&1 | tail -16
