#!/bin/bash
# A/B/C: HEAD~1 tree in .abbase/A/repo, libs .abbase/{B,C}/libstencil_sweep.so with the working tree
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
run() { timeout 300 python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
  python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$2 c$1', round(l['value'],1), round(l['roofline']['frac'],3), l['clocks']['sm_mhz'], l['clocks']['reasons'])"; }
for rep in 1 2; do
for c in $CFGS; do
  (cd .abbase/A/repo && run $c A)
  for v in C; do cp .abbase/$v/libstencil_sweep.so paper_1810_04033_b200/_lib/; run $c $v; done
done
done
