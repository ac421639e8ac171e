#!/bin/bash
# FFMA A/B: BK 8 vs 16, MINB 2 vs 1 (build/exp/libks_minb1.so), on representative FP32 patterns.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/exp_ffma.txt
: > $out
for p in "1 128 128 1" "4 128 128 4" "1 128 128 12" "6 64 64 4" "1 64 64 32" "2 96 96 16" "1 48 48 8" "1 768 192 2" "6 64 64 1"; do
  for lay in bsl bsf; do
    for cfg in "cur:8" "cur:16" "build/exp/libks_minb1.so:8" "build/exp/libks_minb1.so:16"; do
      lib=${cfg%%:*}; [ "$lib" = cur ] && lib=""
      bk=${cfg#*:}
      echo -n "lib=${lib:-cur} bk=$bk " >> $out
      KS_LIB=$lib KS_FFMA_BK=$bk python scripts/run_pattern.py $p --layout $lay --math fp32 --reps 10 >> $out 2>&1
    done
  done
done
