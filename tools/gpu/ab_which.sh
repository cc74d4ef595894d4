set -x
B="python bench.py --steps 10 --warmup 3 --no-sort --c5-copies 0 --c4-layers 0 --leveled-models 0 --ingest-models 0 --no-cpu-baseline"
for L in libxsp_base.so libxsp.so; do
  XSP_LIB=$PWD/paper_1908_06869_b200/lib/$L python -c "import paper_1908_06869_b200._capi as c; print('lib', c.LIB_PATH)"
  XSP_LIB=$PWD/paper_1908_06869_b200/lib/$L timeout 300 $B | python tools/c3line.py
done
