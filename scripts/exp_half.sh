#!/bin/bash
# Half BSL bottleneck experiment: KS_TF32_DEBUG bit 0 skips the epilogue stores.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for dbg in 0 1; do
  for spec in "6 64 64 4 --layout bsl --dtype bf16" "6 64 64 4 --layout bsl --math tf32" "2 128 128 4 --layout bsl --dtype bf16" "6 64 64 4 --layout bsf --dtype bf16" "1 128 128 1 --layout bsf --dtype bf16"; do
    echo "dbg=$dbg $(KS_TF32_DEBUG=$dbg python scripts/run_pattern.py --reps 20 $spec 2>&1 | tail -1)" >> gpurun_out/exp_half.txt
  done
done
