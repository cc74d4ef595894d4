# the N > 1 bench paths on one GPU (2 ranks share it, gloo for the host collectives)
set -x
XSP_DIST_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 4 --warmup 3 --c5-copies 4 --c4-layers 2000000 --leveled-models 16 --ingest-models 6 --no-sort \
  > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err
tail -5 gpurun_out/bench_n2.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench_n2.json'))
print({k: d.get(k) for k in ('value','n_gpus','ms_per_step','scaling')}, 'e2e', d['e2e']['value'])
for k in ('c4','leveled','ingest_jsonl'):
    v=d.get(k) or {}
    print(k, {kk: v.get(kk) for kk in ('value','ms_per_step','combine_ms') if kk in v})
PY
