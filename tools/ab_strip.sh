#!/bin/bash
# A/B of strip2d build variants on config 2: tools/ab_strip.sh "LABEL=EXTRA" ...
mkdir -p gpurun_out
for spec in "$@"; do
  lab=${spec%%=*}; ex=${spec#*=}
  make -s -C paper_1810_04033_b200/csrc clean; make -s -j8 -C paper_1810_04033_b200/csrc EXTRA="$ex" > /dev/null 2>&1
  timeout 300 python -m pytest tests -m gpu -x -q -k "fe9" 2>&1 | tail -1
  for rep in 1 2; do
    timeout 300 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$lab', round(l['value'],1), round(l['roofline']['frac'],3), l['clocks']['sm_mhz'])"
  done
done
make -s -C paper_1810_04033_b200/csrc clean; make -s -j8 -C paper_1810_04033_b200/csrc > /dev/null 2>&1
