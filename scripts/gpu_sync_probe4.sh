mkdir -p gpurun_out
O=gpurun_out/sync_probe4.txt; : > $O
CS=/usr/local/cuda/bin/compute-sanitizer
for c in "1,128,128,12 bsl 240" "2,128,128,1 bsl 240"; do
  echo "### $c" >> $O
  timeout 300 $CS --tool synccheck --print-limit 2 python scripts/sync_probe2.py $c 2>&1 | grep -E "Barrier error|ERROR SUMMARY|done|ks_tf32.cu" | head -6 >> $O
done
timeout 600 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_f32x3.py -q -x > gpurun_out/sync4_pytest.log 2>&1; echo "exit $?" >> gpurun_out/sync4_pytest.log
python scripts/ks_time.py --layout bsl --math tf32 --reps 10 --filter "1,128,128,12;4,128,128,16;16,64,64,4;2,96,96,16;1,64,64,64" --tag oneLane >> $O 2>&1
KS_LIB=paper_2405_15013_b200/lib/libks_base.so python scripts/ks_time.py --layout bsl --math tf32 --reps 10 --filter "1,128,128,12;4,128,128,16;16,64,64,4;2,96,96,16;1,64,64,64" --tag base >> $O 2>&1
