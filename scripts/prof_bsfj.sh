#!/bin/bash
# ncu full-set captures of the TF32 BSF J-gather kernel on representative plans.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
rm -f gpurun_out/prof_*.raw.csv gpurun_out/prof_*.sass.csv.gz
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
ncu_one () {  # name regex args...
  local name=$1; local rx=$2; shift 2
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$rx -s 1 -c 1 -o gpurun_out/prof_$name python scripts/run_pattern.py "$@" --reps 1 > gpurun_out/ncu_$name.log 2>&1
}
for spec in ${SPECS:-"j4g_128_12:1 128 128 12" "j4c_128_4:4 128 128 4" "j3_128_3:1 128 128 3" "j8g_64_32:1 64 64 32" "j2_768_2:1 768 192 2"}; do
  name=${spec%%:*}; p=${spec#*:}
  ncu_one $name ${KREGEX:-ks_tf32_bsfj} $p --layout bsf --math ${MATH:-tf32}
done
for f in gpurun_out/prof_*.ncu-rep; do
  b=${f%.ncu-rep}
  ncu -i $f --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $f --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv
done
rm -f gpurun_out/prof_*.ncu-rep
for spec in ${SPECS:-"j4g_128_12:1 128 128 12" "j4c_128_4:4 128 128 4" "j3_128_3:1 128 128 3" "j8g_64_32:1 64 64 32" "j2_768_2:1 768 192 2"}; do
  p=${spec#*:}
  python scripts/run_pattern.py $p --layout bsf --math ${MATH:-tf32} --reps 20 >> gpurun_out/prof_timing.txt 2>&1
done
