#!/bin/bash
# FD7 iteration: parity (FD7 cases incl. full config 3, slabs), config-3 bench x2, slab geometry of config 3
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fd7 or config3 or slab or windows" 2>&1 | tail -1
for rep in 1 2; do
  timeout 300 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('c3', round(l['value'],1), round(l['roofline']['frac'],3), l['clocks']['sm_mhz'])"
done
timeout 900 python tools/slab_geometry.py --configs 3 > gpurun_out/slab_geometry_c3.json 2> gpurun_out/slab_geometry_c3.err; cat gpurun_out/slab_geometry_c3.err
