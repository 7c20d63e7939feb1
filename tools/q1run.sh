make -s -C paper_1810_04033_b200/csrc >/dev/null; make -s -C oracle
timeout 600 python -m pytest tests -m gpu -x -q -k "fe27q1 or config4 or deterministic or halo" 2>&1 | tail -3
timeout 300 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1
python -c "
import json; l=json.loads(open('gpurun_out/bench_c4.log').read().strip().splitlines()[-1]); print('GLUP/s', l['value'], 'frac', l['roofline']['frac'], l['clocks'])"
python tools/prof_run.py --config 4 --sweeps 1 > gpurun_out/plain4.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k2_q1 -s 0 -c 1 -o gpurun_out/prof_c4v6 -f python tools/prof_run.py --config 4 --sweeps 1 > gpurun_out/ncu4.log 2>&1; tail -1 gpurun_out/ncu4.log
