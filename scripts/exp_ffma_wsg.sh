#!/bin/bash
# FP32 BSF d % 4 == 0: four-j warp-specialised kernel vs the register-staged one (KS_FFMA_WSG=0).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/exp_ffma_wsg.txt
: > $out
for p in "4 128 128 4" "1 128 128 12" "6 64 64 4" "1 64 64 32" "2 96 96 16" "1 48 48 8" "16 48 48 4" "1 64 256 16" "1 256 64 16" "2 48 48 64"; do
  for g in 0 1; do
    echo -n "wsg=$g " >> $out
    KS_FFMA_WSG=$g python scripts/run_pattern.py $p --layout bsf --math fp32 --reps 10 >> $out 2>&1
  done
done
