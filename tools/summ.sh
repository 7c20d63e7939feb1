#!/bin/bash
cd "$(dirname "$0")/.."
tail -n 2 gpurun_out/pytest_gpu.log
for c in 1 2 3 4; do python -c "
import json,sys
try:
  l=json.loads(open('gpurun_out/bench_c$c.log').read().strip().splitlines()[-1])
  print($c, l['config']['workload'], round(l['value'],1), 'GLUP/s', round(l['ms_per_step'],2),'ms', 'frac', round(l['roofline']['frac'],3), l['clocks']['sm_mhz'] if l.get('clocks') else None)
except Exception as e: print($c, 'ERR', open('gpurun_out/bench_c$c.log').read()[-300:])
"; done
