#!/bin/bash
# HEAD state: full GPU suite, smoke, short bench of every config (no CPU legs).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for c in 1 2 3 4 5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/state_c$c.json 2> gpurun_out/state_c$c.err
  python -c "import json;l=json.loads(open('gpurun_out/state_c$c.json').read().strip().splitlines()[-1]);print('c$c', round(l['value'],1), 'GLUP/s', round(l['roofline']['frac'],3), l['roofline'].get('bound'), l['gpu_launches'], l['clocks'])"
done
