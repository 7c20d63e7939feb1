# tools/cfgrun.sh "<pytest -k expr>" "<configs>" [ncu-config] [tag]
# parity subset on the GPU, bench lines for the configs, optional ncu --set full of one config
make -s -C paper_1810_04033_b200/csrc >/dev/null; make -s -C oracle
mkdir -p gpurun_out
if [ -n "$1" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$1" 2>&1 | tail -3; fi
for c in $2; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.log 2>&1
  python -c "
import json; l=json.loads(open('gpurun_out/bench_c$c.log').read().strip().splitlines()[-1]); print('config $c', l['config']['workload'], 'GLUP/s', round(l['value'],1), 'frac', round(l['roofline']['frac'],3), l['clocks']['sm_mhz'])" || tail -5 gpurun_out/bench_c$c.log
done
if [ -n "$3" ]; then
  python tools/prof_run.py --config $3 --sweeps 1 > gpurun_out/plain$3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k[1-4]_ -s 0 -c 1 -f -o gpurun_out/prof_c$3${4} \
      python tools/prof_run.py --config $3 --sweeps 1 > gpurun_out/ncu$3.log 2>&1; tail -1 gpurun_out/ncu$3.log
fi
