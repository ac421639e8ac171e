#!/bin/bash
# Round-2 ncu evidence: bench launch list + full captures of the round-2 kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.raw.csv gpurun_out/prof_*.sass.csv.gz gpurun_out/launches.csv
ncu_one () {  # name regex args...
  local name=$1; local rx=$2; shift 2
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$rx -s 1 -c 1 -o gpurun_out/prof_$name python scripts/run_pattern.py "$@" --reps 1 > gpurun_out/ncu_$name.log 2>&1
}
ncu_one ffma_ws_bsl ks_ffma_ws 2 64 64 16 --layout bsl
ncu_one ffma_wsl_bsf ks_ffma_wsl 1 128 128 16 --layout bsf
ncu_one tf32_bsl_mn ks_tf32_kernel 4 48 48 16 --layout bsl --math tf32
ncu_one tf32_bsl ks_tf32_kernel 1 128 128 16 --layout bsl --math tf32
ncu_one tf32_bsfj ks_tf32_bsfj 1 128 128 16 --layout bsf --math tf32
timeout 300 ncu --set full --import-source on --clock-control none -k regex:fused -c 1 -o gpurun_out/prof_fused_chain python scripts/run_chain.py 12 8192 > gpurun_out/ncu_fused.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sweep --no-verify --no-baselines --no-models \
    > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ks_stream -s 12 -c 3 \
    -o gpurun_out/prof_stream_bench python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-sweep --no-verify --no-baselines --no-models \
    > gpurun_out/ncu_full.log 2>&1
for f in gpurun_out/prof_*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv
done
rm -f gpurun_out/prof_*.ncu-rep
du -sh gpurun_out
