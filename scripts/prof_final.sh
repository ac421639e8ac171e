#!/bin/bash
# ncu captures (full set, one launch each) of every kernel family on representative
# workloads + the bench launch list.  Summaries go to profiles/ via scripts/ncu_summary.py
# and scripts/stall_summary.py.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.raw.csv gpurun_out/prof_*.sass.csv.gz gpurun_out/launches.csv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ncu_one () {  # name regex args...
  local name=$1; local rx=$2; shift 2
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$rx -s 1 -c 1 -o gpurun_out/prof_$name python scripts/run_pattern.py "$@" --reps 1 > gpurun_out/ncu_$name.log 2>&1
}
ncu_one ffma_ws_bsl ks_ffma_ws 6 64 64 4 --layout bsl
ncu_one ffma_ws_bsf1 ks_ffma_ws 64 64 64 1 --layout bsf
ncu_one ffma_rs_bsf ks_ffma_kernel 6 64 64 4 --layout bsf
ncu_one tf32_bsl ks_tf32_kernel 1 128 128 12 --layout bsl --math tf32
ncu_one tf32_bsfj4 ks_tf32_bsfj 4 128 128 4 --layout bsf --math tf32
ncu_one tf32_bsfj_gather ks_tf32_bsfj 1 128 128 12 --layout bsf --math tf32
ncu_one tf32_bsf1 ks_tf32_kernel 64 64 64 1 --layout bsf --math tf32 --B 65536
ncu_one f32x3_bsl ks_tf32_kernel 6 64 64 4 --layout bsl --math f32x3
ncu_one bf16_bsl ks_half_bsl 6 64 64 4 --layout bsl --dtype bf16
ncu_one bf16_bsfj ks_half_bsfj 6 64 64 4 --layout bsf --dtype bf16
timeout 300 ncu --set full --import-source on --clock-control none -k regex:fused -c 1 -o gpurun_out/prof_fused_chain python scripts/run_chain.py 12 8192 > gpurun_out/ncu_fused.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sweep --no-verify --no-baselines \
    > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ks_stream -s 12 -c 3 \
    -o gpurun_out/prof_stream_bench python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-sweep --no-verify --no-baselines \
    > gpurun_out/ncu_full.log 2>&1
# shrink for the 64 MiB copy-back: raw-page CSV + per-line source CSV per capture, then drop the reports
for f in gpurun_out/prof_*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv
done
rm -f gpurun_out/prof_*.ncu-rep
du -sh gpurun_out
