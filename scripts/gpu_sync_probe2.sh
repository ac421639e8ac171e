mkdir -p gpurun_out
O=gpurun_out/sync_probe3.txt; : > $O
CS=/usr/local/cuda/bin/compute-sanitizer
for c in "1,128,128,12 bsl 240" "1,128,128,12 bsl 496" "1,128,128,1 bsf 240" "2,128,128,1 bsl 240" "1,64,64,4 bsl 240"; do
  echo "### $c" >> $O
  timeout 300 $CS --tool synccheck --print-limit 2 python scripts/sync_probe2.py $c 2>&1 | grep -E "Barrier error|ERROR SUMMARY|done|ks_tf32.cu" | head -6 >> $O
done
