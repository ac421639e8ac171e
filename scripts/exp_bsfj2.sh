#!/bin/bash
# TF32 BSF J-kernel epilogue experiments: KS_TF32_DEBUG=4 plain (write-back) stores instead of evict-first.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/exp_bsfj2.txt
: > $out
for p in "4 128 128 4" "1 128 128 12" "1 64 64 32" "2 48 48 16" "1 96 96 24" "16 64 64 4"; do
  for dbg in 0 4; do
    echo -n "dbg=$dbg " >> $out
    KS_TF32_DEBUG=$dbg python scripts/run_pattern.py $p --layout bsf --math tf32 --reps 20 >> $out 2>&1
  done
done
