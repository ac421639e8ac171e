mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cliffs.py tests/test_gpu_random_patterns.py -x -q -k "ffma or cliff or random or tiny or integer" > gpurun_out/ffma2_pytest.log 2>&1; echo "exit $?" >> gpurun_out/ffma2_pytest.log
O=gpurun_out/ffma2_time.jsonl; : > $O
for L in bsl bsf; do
KS_LIB=paper_2405_15013_b200/lib/libks_base.so python scripts/ks_time.py --layout $L --math fp32 --reps 7 --tag base >> $O 2>&1
python scripts/ks_time.py --layout $L --math fp32 --reps 7 --tag ffma2 >> $O 2>&1
done
