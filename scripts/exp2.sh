#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tf32.py -x -q > gpurun_out/pytest_tf32.log 2>&1
tail -3 gpurun_out/pytest_tf32.log > gpurun_out/exp.txt
for spec in "6 64 64 4 --layout bsf --math tf32" "1 128 128 12 --layout bsf --math tf32" "4 96 96 4 --layout bsf --math tf32" "1 64 64 16 --layout bsf --math tf32" "1 48 48 64 --layout bsf --math tf32"; do
  python scripts/run_pattern.py $spec --reps 20 >> gpurun_out/exp.txt 2>&1
done
timeout 900 python bench_sweep.py tf32 > gpurun_out/sweep_tf32.json 2> gpurun_out/sweep_tf32.err
