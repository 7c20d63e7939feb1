#!/bin/bash
# A/B of build variants on one config:  CFG=3 K=fd7 tools/abvar.sh "LABEL=EXTRA" ...
# (each variant: rebuild with EXTRA, GPU tests matching K, two 5-step bench runs)
cd "$(dirname "$0")/.."
CFG=${CFG:-2}; K=${K:-fe9}
mkdir -p gpurun_out
for spec in "$@"; do
  lab=${spec%%=*}; ex=${spec#*=}
  make -s -C paper_1810_04033_b200/csrc clean; make -s -j8 -C paper_1810_04033_b200/csrc EXTRA="$ex" > /dev/null 2>&1
  timeout 600 python -m pytest tests -m gpu -x -q -k "$K" 2>&1 | tail -1
  for rep in 1 2; do
    timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$lab', round(l['value'],1), round(l['roofline']['frac'],3), l['clocks']['sm_mhz'])"
  done
done
make -s -C paper_1810_04033_b200/csrc clean; make -s -j8 -C paper_1810_04033_b200/csrc > /dev/null 2>&1
