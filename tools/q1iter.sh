#!/bin/bash
# Q1 iteration: parity (Q1 cases incl. full config 4), config-4 bench, ncu of one k2_q1col pass.
#   tools/q1iter.sh [label]
cd "$(dirname "$0")/.."
L=${1:-q1}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fe27q1 or q1 or config4" > gpurun_out/pytest_$L.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$L.log
timeout 300 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$L.json 2> gpurun_out/bench_$L.err
python tools/prof_run.py --config 4 --sweeps 2 > gpurun_out/plain_$L.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_q1 -s 1 -c 1 -f \
    -o gpurun_out/prof_$L python tools/prof_run.py --config 4 --sweeps 2 > gpurun_out/ncu_$L.log 2>&1
tail -2 gpurun_out/pytest_$L.log
python -c "import json;l=json.loads(open('gpurun_out/bench_$L.json').read().strip().splitlines()[-1]);print('$L', round(l['value'],1), 'GLUP/s', round(l['roofline']['frac'],3), l['clocks'])"
