#!/bin/bash
# A/B the working tree (current build) against HEAD on a list of configs:
#   tools/abcfg.sh "2 3" "pytest -k expr"
make -s -C paper_1810_04033_b200/csrc > /dev/null 2>&1
mkdir -p gpurun_out
[ -n "$2" ] && timeout 600 python -m pytest tests -m gpu -x -q -k "$2" 2>&1 | tail -1
for c in $1; do
  for rep in 1 2; do
    timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; l=json.loads(sys.stdin.read()); print('new c$c', round(l['value'],1), round(l['roofline']['frac'],3), l['clocks']['sm_mhz'])"
  done
done
if [ -d .abbase ]; then
  cp -r paper_1810_04033_b200/_lib /tmp/_lib_new; rm -rf paper_1810_04033_b200/_lib; cp -r .abbase/_lib paper_1810_04033_b200/_lib
  for c in $1; do
    for rep in 1 2; do
      timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
        python -c "import json,sys; l=json.loads(sys.stdin.read()); print('base c$c', round(l['value'],1), round(l['roofline']['frac'],3), l['clocks']['sm_mhz'])"
    done
  done
fi
