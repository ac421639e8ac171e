#!/bin/bash
# ncu full-set captures of one launch each of the FFMA (BSF, BSL) and TF32 (BSL) kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for spec in "6 64 64 4 --layout bsl --math fp32" "6 64 64 4 --layout bsf --math fp32" "1 128 128 12 --layout bsl --math fp32" \
            "6 64 64 4 --layout bsl --math tf32" "1 128 128 12 --layout bsl --math tf32" "1 128 128 1 --layout bsf --math tf32"; do
  python scripts/run_pattern.py $spec --reps 20 >> gpurun_out/timings.txt 2>&1
done
timeout 300 ncu --set full --import-source on -k regex:ks_ffma -s 1 -c 1 -o gpurun_out/prof_ffma_bsl python scripts/run_pattern.py 6 64 64 4 --layout bsl --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on -k regex:ks_ffma -s 1 -c 1 -o gpurun_out/prof_ffma_bsf python scripts/run_pattern.py 6 64 64 4 --layout bsf --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on -k regex:ks_tf32 -s 1 -c 1 -o gpurun_out/prof_tf32_bsl python scripts/run_pattern.py 6 64 64 4 --layout bsl --math tf32 --reps 1 > /dev/null 2>&1
ls gpurun_out
