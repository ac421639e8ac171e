#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for spec in "6 64 64 4 --layout bsl --math tf32" "1 128 128 12 --layout bsl --math tf32" "4 96 96 4 --layout bsl --math tf32" "1 128 128 1 --layout bsf --math tf32" "64 64 64 1 --layout bsf --math tf32 --B 65536" "1 768 192 2 --layout bsl --math tf32"; do
  python scripts/run_pattern.py $spec --reps 20 >> gpurun_out/exp.txt 2>&1
done
for g in 1 3; do KS_TF32_MAXGRID=$g python tests/multitile_check.py | tail -2 >> gpurun_out/exp.txt; done
timeout 900 python bench_sweep.py tf32 > gpurun_out/sweep_tf32.json 2> gpurun_out/sweep_tf32.err
