#!/bin/bash
# Timings + ncu full-set captures of the half-precision tcgen05 kernels (NEXT-3).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for spec in "6 64 64 4 --layout bsl" "6 64 64 4 --layout bsf" "1 128 128 12 --layout bsl" "1 128 128 1 --layout bsf" \
            "2 64 64 16 --layout bsf" "2 64 64 16 --layout bsl" "6 64 64 4 --layout bsl --math tf32 --dtype f32" \
            "6 64 64 4 --layout bsf --math tf32 --dtype f32" "1 128 128 1 --layout bsf --math tf32 --dtype f32" \
            "2 64 64 16 --layout bsf --math tf32 --dtype f32"; do
  python scripts/run_pattern.py --dtype bf16 --reps 20 $spec >> gpurun_out/timings.txt 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ks_tf32_kernel -s 1 -c 1 -o gpurun_out/prof_bf16_bsl python scripts/run_pattern.py 6 64 64 4 --layout bsl --dtype bf16 --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ks_half_bsfj -s 1 -c 1 -o gpurun_out/prof_bf16_bsfj python scripts/run_pattern.py 6 64 64 4 --layout bsf --dtype bf16 --reps 1 > /dev/null 2>&1
ls gpurun_out
