# A/B of Q1 kernel variants on config 4: tools/q1ab.sh "EXTRA1" "EXTRA2" ...
for v in "$@"; do
  make -s -C paper_1810_04033_b200/csrc clean; make -s -C paper_1810_04033_b200/csrc EXTRA="$v" > /dev/null 2>&1
  timeout 300 python bench.py --config 4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1
  python -c "
import json; l=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('$v', 'GLUP/s', round(l['value'],1), 'frac', round(l['roofline']['frac'],3), l['clocks']['sm_mhz'])" || tail -5 gpurun_out/ab.log
done
make -s -C paper_1810_04033_b200/csrc clean; make -s -C paper_1810_04033_b200/csrc > /dev/null 2>&1
