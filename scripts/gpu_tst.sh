# TF32 J-kernel TMA-store epilogue: parity + A/B timing + role counters
mkdir -p gpurun_out
python -m pytest tests/test_gpu_tf32.py tests/test_gpu_mixed.py tests/test_gpu_bias.py tests/test_gpu_act.py -x -q -k "tf32 or mixed" > gpurun_out/tst_test.txt 2>&1; echo "rc=$?" >> gpurun_out/tst_test.txt
for t in 0 1; do
  KS_TF32_TMASTORE=$t python scripts/ks_time.py --math tf32 --layout bsf --filter dgt1 --tag tst$t >> gpurun_out/tst_time.jsonl 2>&1
  KS_TF32_TMASTORE=$t python scripts/time_factors_io.py --cases "1,64,256,16:65536:bsl:bsf;1,64,256,16:65536:bsf:bsf;1,128,128,4:25088:bsf:bsf;1,768,192,2:25088:bsf:bsf" --tag tst$t >> gpurun_out/tst_io.jsonl 2>&1
  KS_TF32_TMASTORE=$t python scripts/prof_roles.py "1,128,128,32:25088:bsf:bsf;1,64,256,16:65536:bsl:bsf;1,96,96,16:25088:bsf:bsf" > gpurun_out/tst_roles_$t.txt 2>&1
done
python -m pytest tests/test_gpu_sweep_full.py -x -q -k "tf32" >> gpurun_out/tst_test.txt 2>&1; echo "rc2=$?" >> gpurun_out/tst_test.txt
