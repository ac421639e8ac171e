#!/bin/bash
# FFMA warp-specialised kernel vs the register-staged one (KS_FFMA_WS=0), FP32 patterns, both layouts.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/exp_ffma_ws.txt
: > $out
for p in ${PATS:-"1 128 128 1" "4 128 128 4" "1 128 128 12" "6 64 64 4" "1 64 64 32" "2 96 96 16" "1 768 192 2" "6 64 64 1" "64 64 64 1" "1 96 96 1"}; do
  for lay in bsl bsf; do
    for ws in 0 1; do
      echo -n "ws=$ws " >> $out
      KS_FFMA_WS=$ws python scripts/run_pattern.py $p --layout $lay --math fp32 --reps 10 >> $out 2>&1
    done
  done
done
