#!/bin/bash
# One GPU iteration: parity tests, bench of every config, optional ncu of one config.
#   tools/gpu_iter.sh [ncu-config ...]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 2 3 4 1; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.log 2>&1
done
for c in "$@"; do
  python tools/prof_run.py --config $c --sweeps 2 > gpurun_out/plain$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k[1-4]_ -s 1 -c 1 \
      -o gpurun_out/prof_c$c python tools/prof_run.py --config $c --sweeps 2 > gpurun_out/ncu$c.log 2>&1
done
tail -n 2 gpurun_out/pytest_gpu.log
