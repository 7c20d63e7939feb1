#!/bin/bash
# End-of-round check: GPU parity suite, smoke(), the driver's default bench line,
# config-4 bench + ncu --set full of its kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
(nproc; free -g; nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv) > gpurun_out/host.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/default.json 2> gpurun_out/default.err
timeout 900 python bench.py --impl reference > gpurun_out/ref_default.json 2> gpurun_out/ref_default.err
python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/l4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_c4.csv python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncul4.log 2>&1
python tools/prof_run.py --config 4 --sweeps 2 > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_ -s 1 -c 1 -f \
    -o gpurun_out/prof_c4 python tools/prof_run.py --config 4 --sweeps 2 > gpurun_out/ncu4.log 2>&1
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -1
