#!/bin/bash
# Race evidence without compute-sanitizer (closed on this pool): the bitwise GPU
# parity suite under the timing-perturbation build (-DSL_FUZZ, common.cuh), several
# rounds (delays are clock-seeded, so every round is a different interleaving), then
# three negative controls (-DSL_FUZZ_BREAK=n: 1 drops a block barrier of k2_q1col, 2 the mbarrier wait of
# k2_strip2d's row slots, 3 the per-step block barrier of k2_col3d_fd7) that must fail.
#   tools/fuzz_race.sh [rounds]
cd "$(dirname "$0")/.."
R=${1:-10}
mkdir -p gpurun_out
OUT=gpurun_out/fuzz_race.txt
: > $OUT
build() { make -s -C paper_1810_04033_b200/csrc clean; make -s -j8 -C paper_1810_04033_b200/csrc EXTRA="$1" > gpurun_out/fuzz_build.log 2>&1 || { echo "BUILD FAILED $1" | tee -a $OUT; tail -5 gpurun_out/fuzz_build.log; exit 1; }; }
SEL='not config4 and not config2_fe9_8194 and not config3'
build "-DSL_FUZZ"
for r in $(seq 1 $R); do
  t0=$(date +%s)
  res=$(timeout 3000 python -m pytest tests -m gpu -q -k "$SEL" 2>&1 | tail -1)
  echo "fuzz round $r: $res ($(( $(date +%s) - t0 )) s)" | tee -a $OUT
done
res=$(timeout 1800 python -m pytest tests -m gpu -q -k "config4 or config2_fe9_8194 or config3" 2>&1 | tail -1)
echo "fuzz full-size configs 2-4: $res" | tee -a $OUT
for b in 1 2 3; do
  build "-DSL_FUZZ -DSL_FUZZ_BREAK=$b"
  case $b in 1) k="fe27q1 or q1";; 2) k="fe9";; 3) k="fd7";; esac
  res=$(timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$k" 2>&1 | grep -E "passed|failed" | tail -1)
  echo "negative control $b ($k): $res" | tee -a $OUT
done
build ""
res=$(timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "small_and_ragged" 2>&1 | tail -1)
echo "plain rebuild: $res" | tee -a $OUT
