#!/bin/bash
# A/B of the TMA L2 promotion mode on configs 4 and 3 (bench + DRAM bytes per launch via ncu metrics)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in "p128=-DSL_TMAP_PROMO=CU_TENSOR_MAP_L2_PROMOTION_L2_128B" "pnone=-DSL_TMAP_PROMO=CU_TENSOR_MAP_L2_PROMOTION_NONE" "p256="; do
  lab=${spec%%=*}; ex=${spec#*=}
  touch paper_1810_04033_b200/csrc/k2_fused.cu
  make -s -j8 -C paper_1810_04033_b200/csrc EXTRA="$ex" > gpurun_out/build_$lab.log 2>&1 || { echo "$lab BUILD FAILED"; continue; }
  timeout 300 python -m pytest tests -m gpu -x -q -k "small_and_ragged and (fe27q1 or fd7)" 2>&1 | tail -1
  for c in 4 3; do
    for rep in 1 2; do
      timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$lab c$c', round(l['value'],1), round(l['roofline']['frac'],3), l['clocks']['sm_mhz'])"
    done
    timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k2_ -s 1 -c 1 python tools/prof_run.py --config $c --sweeps 2 2>/dev/null | grep -E "dram__bytes" | tr -s ' ' | tr '\n' ';'; echo
  done
done
