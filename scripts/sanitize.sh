#!/bin/bash
# compute-sanitizer gate (SURVEY §4 layer 8): memcheck, racecheck, synccheck over
# every kernel family at small shapes (scripts/sanitize_driver.py), once with the
# default grid and once with KS_TF32_MAXGRID=2 (persistent CTAs wrap their
# TMA / mbarrier / TMEM rings).  Logs under gpurun_out/sanitize/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for grid in 0 2; do
    log=gpurun_out/sanitize/${tool}_grid${grid}.txt
    extra=""
    # (no --leak-check: the chain workspace pool keeps its blocks for the process lifetime by design)
    KS_TF32_MAXGRID=$grid timeout 1200 $CS --tool $tool $extra --print-limit 20 \
      python scripts/sanitize_driver.py > $log 2>&1
    echo "exit $?" >> $log
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|exit" $log | tail -3
  done
done
