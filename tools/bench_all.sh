#!/bin/bash
# Full bench line for every BASELINE config + ncu launch lists (round artefacts).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c > gpurun_out/full_c$c.json 2> gpurun_out/full_c$c.err
done
timeout 600 python bench.py --impl reference > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err
for c in 1 2 3 4 5; do
  python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/l$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_c$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncul$c.log 2>&1
done
ls gpurun_out
