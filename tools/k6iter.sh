#!/bin/bash
# K6 iteration: FD5 parity (small/ragged, config 1 full, pipeline, verify), config-1 bench, ncu of k6.
cd "$(dirname "$0")/.."
L=${1:-k6}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fd5 or config1 or pipeline or verify" > gpurun_out/pytest_$L.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_$L.log
tail -3 gpurun_out/pytest_$L.log
for rep in 1 2; do
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$L.json 2> gpurun_out/bench_$L.err
python -c "import json;l=json.loads(open('gpurun_out/bench_$L.json').read().strip().splitlines()[-1]);print('$L', round(l['value'],1), 'GLUP/s', round(l['ms_per_step'],4), 'ms', l['gpu_launches'], l['clocks'])"
done
python tools/prof_run.py --config 1 --sweeps 100 > gpurun_out/plain_$L.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k6_ -s 0 -c 1 -f \
    -o gpurun_out/prof_$L python tools/prof_run.py --config 1 --sweeps 100 > gpurun_out/ncu_$L.log 2>&1
tail -1 gpurun_out/ncu_$L.log
