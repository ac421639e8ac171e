mkdir -p gpurun_out
KS_FFMA_WSL=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_patterns.py tests/test_gpu_bias.py tests/test_gpu_sweep_full.py -x -q -k "ffma or random or bias or integer or fp32" > gpurun_out/wsl_pytest.log 2>&1; echo "exit $?" >> gpurun_out/wsl_pytest.log
O=gpurun_out/wsl_time.jsonl; : > $O
python scripts/ks_time.py --layout bsf --math fp32 --reps 7 --filter dgt1 --tag base >> $O 2>&1
KS_FFMA_WSL=1 python scripts/ks_time.py --layout bsf --math fp32 --reps 7 --filter dgt1 --tag wsl >> $O 2>&1
