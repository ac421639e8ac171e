mkdir -p gpurun_out
python -m pytest tests/test_gpu_tf32.py tests/test_gpu_mixed.py tests/test_gpu_tf32_dense.py -x -q > gpurun_out/bn256d_test.txt 2>&1; echo "rc=$?" >> gpurun_out/bn256d_test.txt
C="1,768,192,2:25088:bsf:bsf;1,128,128,2:25088:bsf:bsf;1,128,128,4:25088:bsf:bsf;2,128,128,2:25088:bsf:bsf;1,1536,384,1:25088:bsf:bsf"
for t in 0 1; do KS_TF32_BN256D=$t python scripts/time_factors_io.py --cases "$C" --tag w$t >> gpurun_out/bn256d.jsonl 2>&1; done
for t in 0 1; do KS_TF32_BN256D=$t python scripts/time_models.py --reps 20 --tag w$t --only vit_up >> gpurun_out/bn256d.jsonl 2>&1; done
