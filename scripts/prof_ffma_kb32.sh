#!/bin/bash
# ncu full-set captures of the TMA-fed FFMA kernel on a b = 96 BSL pattern, 32 vs 16 l per chunk.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.raw.csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for kb in 1 0; do
  KS_FFMA_KB32=$kb timeout 300 ncu --set full --import-source on --clock-control none -k regex:ks_ffma_ws -s 1 -c 1 \
    -o gpurun_out/prof_kb32_$kb python scripts/run_pattern.py 2 96 96 16 --layout bsl --reps 1 > gpurun_out/ncu_kb32_$kb.log 2>&1
  ncu -i gpurun_out/prof_kb32_$kb.ncu-rep --page raw --csv > gpurun_out/prof_kb32_$kb.raw.csv 2>/dev/null
done
rm -f gpurun_out/prof_*.ncu-rep
