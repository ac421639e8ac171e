mkdir -p gpurun_out
python -m pytest tests/test_gpu_tf32.py tests/test_gpu_mixed.py tests/test_gpu_bias.py tests/test_gpu_act.py tests/test_gpu_sweep_full.py -x -q -k "tf32 or mixed" > gpurun_out/tstd_test.txt 2>&1; echo "rc=$?" >> gpurun_out/tstd_test.txt
for g in 1 3; do KS_TF32_MAXGRID=$g python tests/multitile_check.py >> gpurun_out/tstd_test.txt 2>&1; echo "mt rc=$?" >> gpurun_out/tstd_test.txt; done
C="64,64,64,1:65536:bsl:bsf;64,64,64,1:65536:bsf:bsf;6,64,64,1:25088:bsf:bsf;6,64,256,1:25088:bsf:bsf;16,128,128,1:25088:bsf:bsf;1,128,128,1:25088:bsf:bsf;4,64,64,1:25088:bsl:bsf"
for t in 0 1; do KS_TF32_TMASTORE=$t python scripts/time_factors_io.py --cases "$C" --tag t$t >> gpurun_out/tstd_io.jsonl 2>&1; done
for t in 0 1; do KS_TF32_TMASTORE=$t python scripts/ks_time.py --math tf32 --layout bsf --filter d1 --tag t$t >> gpurun_out/tstd_io.jsonl 2>&1; done
python scripts/time_models.py --reps 20 --tag tstd > gpurun_out/tstd_models.jsonl 2>&1
