#!/bin/bash
# Half BSL (swap-AB) experiment: tile width KS_HB_NT and batch size.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for nt in 128 256; do
  for spec in "6 64 64 4 --layout bsl --dtype bf16" "2 128 128 4 --layout bsl --dtype bf16" "6 64 64 4 --layout bsl --dtype bf16 --B 100352" "2 128 128 4 --layout bsl --dtype bf16 --B 100352" "6 64 64 4 --layout bsl --math tf32 --B 100352"; do
    echo "nt=$nt $(KS_HB_NT=$nt python scripts/run_pattern.py --reps 20 $spec 2>&1 | tail -1)" >> gpurun_out/exp_hb.txt
  done
done
