#!/bin/bash
# FFMA warp-specialised kernels vs the register-staged one (KS_FFMA_WS=0), FP32 patterns.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/exp_ffma_ws.txt
: > $out
for p in ${PATS:-"4 128 128 4" "1 128 128 12" "6 64 64 4" "1 64 64 32" "2 96 96 16" "1 768 192 2" "1 48 48 8" "16 48 48 4" "1 64 256 16" "1 256 64 16" "1 128 128 2"}; do
  for lay in ${LAYS:-bsf}; do
    for ws in 0 1; do
      echo -n "ws=$ws " >> $out
      KS_FFMA_WS=$ws python scripts/run_pattern.py $p --layout $lay --math fp32 --reps 10 >> $out 2>&1
    done
  done
done
