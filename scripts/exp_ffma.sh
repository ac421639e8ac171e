#!/bin/bash
# FFMA experiment timings (FP32 CUDA-core kernel) on representative sweep patterns.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for spec in "6 64 64 4 --layout bsl" "6 64 64 4 --layout bsf" "1 128 128 12 --layout bsl" "1 128 128 12 --layout bsf" "2 48 48 16 --layout bsf" "4 96 96 2 --layout bsf" "64 64 64 1 --layout bsf" "1 48 48 3 --layout bsf"; do
  echo "${TAG:-x} $(python scripts/run_pattern.py --reps 20 $spec 2>&1 | tail -1)" >> gpurun_out/exp_ffma.txt
done
