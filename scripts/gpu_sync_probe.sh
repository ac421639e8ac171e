mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
o=gpurun_out/sanitize/sync_probe.txt; rm -f $o
for env in "X=1" "KS_PDL=0" "KS_TF32_MAXGRID=1"; do
 for case in "1,128,128,12 260" "1,128,128,12 128" "1,64,64,32 260" "1,128,128,1 1024" "1,96,96,8 1024"; do
  echo "### $env $case" >> $o
  env $env timeout 300 $CS --tool synccheck --print-limit 2 python scripts/sync_probe.py $case 2>&1 | grep -E "ERROR SUMMARY|done|Missing|at void" | head -4 >> $o
 done
done
