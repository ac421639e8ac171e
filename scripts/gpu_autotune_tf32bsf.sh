mkdir -p gpurun_out
python -m pytest tests/test_gpu_tf32.py tests/test_gpu_mixed.py -x -q -k "tf32 or mixed" > gpurun_out/at_test.txt 2>&1; echo "rc=$?" >> gpurun_out/at_test.txt
timeout 2400 python scripts/autotune.py --out gpurun_out/autotune_tf32_bsf_v2.json --only tf32:bsf --reps 10 > gpurun_out/autotune_tf32_bsf_v2.log 2>&1
echo "exit $?" >> gpurun_out/autotune_tf32_bsf_v2.log
