#!/bin/bash
# A/B timing of TF32 BSF J-gather variants (KS_LIB = alternative build) and debug knobs.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/exp_bsfj.txt
: > $out
for p in ${PATS:-"1 768 192 2" "4 128 128 4" "1 128 128 12" "1 64 64 32" "1 128 128 3" "4 64 64 4" "1 96 96 6" "2 48 48 16"}; do
  for cfg in ${CFGS:-"cur:0" "cur:1" "build/exp/libks_v6.so:0"}; do
    lib=${cfg%%:*}; [ "$lib" = cur ] && lib=""
    dbg=${cfg#*:}
    echo -n "lib=${lib:-cur} dbg=$dbg " >> $out
    KS_LIB=$lib KS_TF32_DEBUG=$dbg python scripts/run_pattern.py $p --layout bsf --math ${MATH:-tf32} --reps 20 >> $out 2>&1
  done
done
