#!/bin/bash
# cluster-pair variant of k2_q1col: build, small parity first (short timeout: a wrong barrier count hangs), then the rest
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
touch paper_1810_04033_b200/csrc/k2_q1col.cuh
make -s -j8 -C paper_1810_04033_b200/csrc EXTRA="-DQ1_CLUSTER=1" > gpurun_out/build_cl.log 2>&1 || { echo BUILD FAILED; tail -5 gpurun_out/build_cl.log; exit 1; }
timeout 120 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "small_and_ragged and fe27q1" 2>&1 | tail -3
[ ${PIPESTATUS[0]} -ne 0 ] && { echo "small parity failed or hung"; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q -k "fe27q1 or q1 or config4" 2>&1 | tail -2
for rep in 1 2; do
  timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('cl', round(l['value'],1), round(l['roofline']['frac'],3), l['clocks']['sm_mhz'], l['clocks']['reasons'])"
done
touch paper_1810_04033_b200/csrc/k2_q1col.cuh
make -s -j8 -C paper_1810_04033_b200/csrc > gpurun_out/build_plain.log 2>&1
for rep in 1 2; do
  timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('default', round(l['value'],1), round(l['roofline']['frac'],3), l['clocks']['sm_mhz'], l['clocks']['reasons'])"
done
