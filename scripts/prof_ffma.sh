#!/bin/bash
# ncu full-set captures of the FP32 FFMA kernels (warp-specialised and register-staged).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.raw.csv gpurun_out/prof_*.sass.csv.gz
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ncu_one () {  # name regex args...
  local name=$1; local rx=$2; shift 2
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$rx -s 1 -c 1 -o gpurun_out/prof_$name python scripts/run_pattern.py "$@" --reps 1 > gpurun_out/ncu_$name.log 2>&1
}
ncu_one ws_bsl ks_ffma_ws 4 128 128 4 --layout bsl
ncu_one ws_bsf1 ks_ffma_ws 64 64 64 1 --layout bsf
ncu_one rs_bsf4 ks_ffma_kernel 4 128 128 4 --layout bsf
for f in gpurun_out/prof_*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv
done
rm -f gpurun_out/prof_*.ncu-rep
