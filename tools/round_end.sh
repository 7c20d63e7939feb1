#!/bin/bash
# Round artefacts: full bench lines + launch lists (bench_all.sh), then one
# ncu --set full capture of the dominant kernel of configs 2, 3, 4.
cd "$(dirname "$0")/.."
bash tools/bench_all.sh
for c in 2 3 4; do
  python tools/prof_run.py --config $c --sweeps 2 > gpurun_out/plain$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k2_ -s 1 -c 1 -f \
      -o gpurun_out/prof_c$c python tools/prof_run.py --config $c --sweeps 2 > gpurun_out/ncu$c.log 2>&1
  tail -1 gpurun_out/ncu$c.log
done
