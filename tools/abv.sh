#!/bin/bash
# A/B of prebuilt library variants .abbase/<V>/libstencil_sweep.so on configs $CFGS:
#   CFGS="4" PYK="fe27q1" tools/abv.sh B C
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cp paper_1810_04033_b200/_lib/libstencil_sweep.so /tmp/_lib_keep.so
for v in "$@"; do
  cp .abbase/$v/libstencil_sweep.so paper_1810_04033_b200/_lib/
  [ -n "$PYK" ] && echo "[$v] $(timeout 600 python -m pytest tests -m gpu -x -q -k "$PYK" 2>&1 | tail -1)"
done
for rep in 1 2; do for c in $CFGS; do for v in "$@"; do
  cp .abbase/$v/libstencil_sweep.so paper_1810_04033_b200/_lib/
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; l=json.loads(sys.stdin.read()); print('[$v] c$c', round(l['value'],1), round(l['roofline']['frac'],3), l['clocks']['sm_mhz'], l['clocks']['reasons'])"
done; done; done
cp /tmp/_lib_keep.so paper_1810_04033_b200/_lib/libstencil_sweep.so
