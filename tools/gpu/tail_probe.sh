set -x
for t in 1000000 3000000 6000000 12000000; do XSP_TAIL_SPANS=$t timeout 600 python tools/e2e_packed_probe.py 12000000 2>&1 | grep "packed:\|done\|chunk [0-9] spans" | head -12; done
