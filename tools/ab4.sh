#!/bin/bash
# A/B of build variants on config 4 with the Q1 parity subset: tools/ab4.sh "EXTRA1" "EXTRA2" ...
mkdir -p gpurun_out
for v in "$@"; do
  make -s -C paper_1810_04033_b200/csrc clean; make -s -C paper_1810_04033_b200/csrc EXTRA="$v" > /dev/null 2>&1
  timeout 300 python -m pytest tests -m gpu -x -q -k "fe27q1" 2>&1 | tail -1
  for rep in 1 2; do
    timeout 300 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1
    python -c "
import json; l=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('[$v]', 'GLUP/s', round(l['value'],1), 'ms', round(l['ms_per_step'],2), l['clocks']['sm_mhz'])" || tail -3 gpurun_out/ab.log
  done
done
make -s -C paper_1810_04033_b200/csrc clean; make -s -C paper_1810_04033_b200/csrc > /dev/null 2>&1
