#!/bin/bash
# compute-sanitizer racecheck + synccheck (+ memcheck) over every sweep kernel
# on small grids (tools/race_run.py); logs to gpurun_out/sanitize_*.log.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for c in ${CASES:-strip2d fd5strip block2d resident col3d q1col stream3d patch k1 lex peer}; do
  for tool in racecheck synccheck memcheck; do
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $extra --print-limit 50 python tools/race_run.py $c \
        > gpurun_out/sanitize_${tool}_$c.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_${tool}_$c.log | tail -1)"
  done
done | tee gpurun_out/sanitize_summary.txt
