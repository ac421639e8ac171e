mkdir -p gpurun_out
KS_TF32_MN=1 timeout 900 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_mixed.py -x -q -k "bsl or lf" > gpurun_out/mn_pytest.log 2>&1; echo "exit $?" >> gpurun_out/mn_pytest.log
python scripts/ks_time.py --layout bsl --math tf32 --reps 10 --tag v1 > gpurun_out/mn_time.jsonl 2>&1
KS_TF32_MN=1 python scripts/ks_time.py --layout bsl --math tf32 --reps 10 --tag mn >> gpurun_out/mn_time.jsonl 2>&1
