mkdir -p gpurun_out
python -m pytest tests/test_gpu_mixed.py tests/test_gpu_tf32.py -x -q > gpurun_out/mnj_test.txt 2>&1; echo "rc=$?" >> gpurun_out/mnj_test.txt
C="1,64,256,16:65536:bsl:bsf;1,64,64,16:25088:bsl:bsf;1,128,128,16:25088:bsl:bsf;1,48,48,32:25088:bsl:bsf;1,96,96,8:25088:bsl:bsf;2,64,64,4:25088:bsl:bsf;1,128,128,32:25088:bsl:bsf"
for m in 0 1; do KS_TF32_MNJ=$m python scripts/time_factors_io.py --cases "$C" --tag mnj$m >> gpurun_out/mnj_time.jsonl 2>&1; done
python scripts/time_models.py --reps 20 --tag mnj > gpurun_out/mnj_models.jsonl 2>&1
