mkdir -p gpurun_out
python -m pytest tests/test_gpu_tf32.py tests/test_gpu_mixed.py tests/test_gpu_sweep_full.py -x -q -k "tf32 or mixed" > gpurun_out/fill_test.txt 2>&1; echo "rc=$?" >> gpurun_out/fill_test.txt
C="1,128,128,3:25088:bsf:bsf;1,96,96,3:25088:bsf:bsf;1,128,128,2:25088:bsf:bsf;1,64,64,3:25088:bsf:bsf;1,128,128,4:25088:bsf:bsf;1,768,192,2:25088:bsf:bsf;2,128,128,2:25088:bsf:bsf;1,128,128,6:25088:bsf:bsf"
for f in 0 1 0 1; do KS_TF32_BSFJ_FILL=$f python scripts/time_factors_io.py --cases "$C" --tag f$f >> gpurun_out/fill_time.jsonl 2>&1; done
for f in 0 1; do KS_TF32_BSFJ_FILL=$f python scripts/time_models.py --reps 20 --tag f$f --only vit_down,vit_up >> gpurun_out/fill_time.jsonl 2>&1; done
