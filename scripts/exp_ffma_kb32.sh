#!/bin/bash
# FFMA warp-specialised kernel, BSL b = 96: 32 l per staged chunk (default) vs 16 (KS_FFMA_KB32=0).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/exp_ffma_kb32.txt
: > $out
for p in ${PATS:-"2 96 96 16" "1 96 96 32" "4 96 96 4" "1 96 192 8" "1 96 64 16" "16 96 96 1" "1 192 96 16"}; do
  for kb in 0 1; do
    echo -n "kb32=$kb " >> $out
    KS_FFMA_KB32=$kb python scripts/run_pattern.py $p --layout bsl --math fp32 --reps 10 >> $out 2>&1
  done
done
