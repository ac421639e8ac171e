# TF32 J-kernel: 4 vs 8 epilogue warps -- parity, role counters, A/B timing
mkdir -p gpurun_out
python -m pytest tests/test_gpu_tf32.py tests/test_gpu_mixed.py tests/test_gpu_sweep_full.py -x -q -k "tf32 or mixed" > gpurun_out/ew_test.txt 2>&1; echo "rc=$?" >> gpurun_out/ew_test.txt
for ew in 4 8; do
  KS_TF32_EW=$ew python scripts/prof_roles.py "1,128,128,32:25088:bsf:bsf;1,64,256,16:65536:bsl:bsf;1,256,64,16:65536:bsf:bsl;1,96,96,16:25088:bsf:bsf" > gpurun_out/ew_roles_$ew.txt 2>&1
  KS_TF32_EW=$ew python scripts/ks_time.py --math tf32 --layout bsf --filter dgt1 --tag ew$ew >> gpurun_out/ew_time.jsonl 2>&1
  KS_TF32_EW=$ew python scripts/time_factors_io.py --cases "1,64,256,16:65536:bsl:bsf;1,256,64,16:65536:bsf:bsl;1,64,256,16:65536:bsf:bsf;1,128,128,3:25088:bsf:bsf;1,768,192,2:25088:bsf:bsf" --tag ew$ew >> gpurun_out/ew_io.jsonl 2>&1
done
