#!/bin/bash
# A/B of k2_q1col build variants:  tools/q1ab.sh "LABEL=EXTRA" ...
# (each: rebuild, Q1 parity tests, two 5-step config-4 bench runs; labels listed in NCU="a b" get an ncu capture)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in "$@"; do
  lab=${spec%%=*}; ex=${spec#*=}
  touch paper_1810_04033_b200/csrc/k2_q1col.cuh
  make -s -j8 -C paper_1810_04033_b200/csrc EXTRA="$ex" > gpurun_out/build_$lab.log 2>&1 || { echo "$lab BUILD FAILED"; tail -5 gpurun_out/build_$lab.log; continue; }
  grep -A2 "k2_q1colILi1ELb0ELi2ELb0" paper_1810_04033_b200/_lib/obj/k2_fused.ptxas.txt | grep -E "registers|spill" | tr '\n' ' '; echo
  timeout 600 python -m pytest tests -m gpu -x -q -k "fe27q1 or q1 or config4" 2>&1 | tail -1
  for rep in 1 2; do
    timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$lab', round(l['value'],1), round(l['roofline']['frac'],3), l['clocks']['sm_mhz'], l['clocks']['reasons'])"
  done
  if [[ " $NCU " == *" $lab "* ]]; then
    python tools/prof_run.py --config 4 --sweeps 2 > /dev/null 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:k2_q1 -s 1 -c 1 -f \
      -o gpurun_out/prof_$lab python tools/prof_run.py --config 4 --sweeps 2 > gpurun_out/ncu_$lab.log 2>&1
  fi
done
