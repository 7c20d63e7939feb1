#!/bin/bash
# A/B of kernel build variants on one config: tools/ab2.sh CONFIG "EXTRA1" "EXTRA2" ...
c=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  make -s -C paper_1810_04033_b200/csrc clean; make -s -C paper_1810_04033_b200/csrc EXTRA="$v" > /dev/null 2>&1
  timeout 300 python -m pytest tests -m gpu -x -q -k "fe9 or fd5" 2>&1 | tail -1
  for rep in 1 2; do
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1
    python -c "
import json; l=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('[$v]', 'GLUP/s', round(l['value'],1), 'frac', round(l['roofline']['frac'],3), l['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.log
  done
done
make -s -C paper_1810_04033_b200/csrc clean; make -s -C paper_1810_04033_b200/csrc > /dev/null 2>&1
