#!/bin/bash
# Round-2 artefacts at HEAD: full bench line of every BASELINE config (+ the reference arm of the
# default config), ncu launch lists with per-launch DRAM bytes, one ncu --set full capture of each
# dominant kernel summarised on the box (tools/ncu_brief.py), slab-geometry compute rates.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out
(nproc; free -g | head -2; grep -m1 "model name" /proc/cpuinfo; nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv) > $O/host.txt 2>&1
for c in ${CONFIGS:-4 1 2 3 5}; do
  timeout 900 python bench.py --config $c > $O/bench_c$c.json 2> $O/bench_c$c.err
done
[ -z "$CONFIGS" ] && timeout 900 python bench.py --impl reference > $O/bench_reference_c4.json 2> $O/bench_reference_c4.err
for c in ${CONFIGS:-1 2 3 4 5}; do
  python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/l$c.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $O/launches_c$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncul$c.log 2>&1
done
declare -A KERN=([1]=k6_ [2]=k2_strip2d [3]=k2_col3d [4]=k2_q1col [5]=k3_patch)
declare -A SW=([1]=100 [2]=4 [3]=2 [4]=2 [5]=200)
declare -A SKIP=([1]=0 [2]=1 [3]=1 [4]=1 [5]=0)
declare -A PTS=([1]=104857600 [2]=134217728 [3]=134217728 [4]=1073741824 [5]=3355443200)
for c in ${CONFIGS:-1 2 3 4 5}; do
  python tools/prof_run.py --config $c --sweeps ${SW[$c]} > $O/plain$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KERN[$c]} -s ${SKIP[$c]} -c 1 -f \
      -o $O/prof_c$c python tools/prof_run.py --config $c --sweeps ${SW[$c]} > $O/ncu$c.log 2>&1
  python tools/ncu_brief.py $O/prof_c$c.ncu-rep ${PTS[$c]} > $O/ncu_full_c$c.txt 2>&1
  [ $c != 4 ] && rm -f $O/prof_c$c.ncu-rep
  tail -3 $O/ncu_full_c$c.txt
done
[ -z "$CONFIGS" ] && { timeout 1200 python tools/slab_geometry.py > $O/slab_geometry.json 2> $O/slab_geometry.err; tail -20 $O/slab_geometry.err; }
for c in ${CONFIGS:-4 1 2 3 5}; do python -c "
import json
l=json.loads(open('$O/bench_c$c.json').read().strip().splitlines()[-1])
print('c$c', round(l['value'],1), round(l['roofline']['frac'],3), l['roofline']['bound'], 'e2e', round(l['e2e']['value'],1), 'cpu', round(l['cpu_baseline']['value'],2), l['clocks'])
"; done
