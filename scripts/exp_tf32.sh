#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for dbg in 0 1 2 3; do
  for spec in "6 64 64 4 --layout bsl --math tf32" "1 128 128 12 --layout bsl --math tf32" "1 128 128 1 --layout bsf --math tf32"; do
    echo "dbg=$dbg $(KS_TF32_DEBUG=$dbg python scripts/run_pattern.py $spec --reps 20 2>&1)" >> gpurun_out/exp.txt
  done
done
for spec in "6 64 64 4 --layout bsf" "1 128 128 12 --layout bsf" "4 96 96 4 --layout bsf" "1 64 64 2 --layout bsf" "1 48 48 3 --layout bsf"; do
  python scripts/run_pattern.py $spec --reps 20 >> gpurun_out/exp.txt 2>&1
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ffma or sweep" > gpurun_out/pytest_ffma.log 2>&1
tail -2 gpurun_out/pytest_ffma.log >> gpurun_out/exp.txt
