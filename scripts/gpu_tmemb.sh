mkdir -p gpurun_out
python -m pytest tests/test_gpu_tf32.py tests/test_gpu_mixed.py tests/test_gpu_bias.py tests/test_gpu_act.py tests/test_gpu_sweep_full.py tests/test_gpu_f32x3.py -x -q -k "tf32 or mixed or f32x3" > gpurun_out/tmemb_test.txt 2>&1; echo "rc=$?" >> gpurun_out/tmemb_test.txt
for g in 1 3; do KS_TF32_MAXGRID=$g python tests/multitile_check.py >> gpurun_out/tmemb_test.txt 2>&1; echo "mt rc=$?" >> gpurun_out/tmemb_test.txt; done
python scripts/ks_time.py --math tf32 --layout bsf --filter dgt1 --tag tmemb > gpurun_out/tmemb_time.jsonl 2>&1
python scripts/time_factors_io.py --cases "1,64,256,16:65536:bsl:bsf;1,256,64,16:65536:bsf:bsl;1,256,64,16:65536:bsf:bsf;1,128,128,3:25088:bsf:bsf" --tag tmemb >> gpurun_out/tmemb_time.jsonl 2>&1
python scripts/prof_roles.py "1,128,128,32:25088:bsf:bsf;1,96,96,16:25088:bsf:bsf" > gpurun_out/tmemb_roles.txt 2>&1
