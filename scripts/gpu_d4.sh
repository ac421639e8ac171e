mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ffma_wsl.py tests/test_gpu_sweep_full.py -q -x -k "wsl or (fp32 and bsf)" > gpurun_out/d4_pytest.log 2>&1; echo "exit $?" >> gpurun_out/d4_pytest.log
C="1,48,48,4;2,48,48,4;6,48,48,4;16,48,48,4;1,64,64,4;4,64,64,4;16,64,64,4;1,96,96,4;8,96,96,4;1,128,128,4;16,128,128,4"
O=gpurun_out/d4_time.jsonl; : > $O
KS_LIB=paper_2405_15013_b200/lib/libks_base.so python scripts/ks_time.py --layout bsf --math fp32 --reps 10 --filter "$C" --tag base >> $O 2>&1
python scripts/ks_time.py --layout bsf --math fp32 --reps 10 --filter "$C" --tag box2d >> $O 2>&1
