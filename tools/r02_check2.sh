cd /root/repo
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "small_and_ragged or replaced_rhs or nonfinite" > gpurun_out/pytest_stream.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stream.log
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/fp64_peak.cu -o /tmp/fp64_peak && /tmp/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 2400 bash tools/sanitize.sh > gpurun_out/sanitize_run.log 2>&1
tail -3 gpurun_out/pytest_stream.log
