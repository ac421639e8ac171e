mkdir -p gpurun_out
python -m pytest tests/test_gpu_tf32.py tests/test_gpu_mixed.py tests/test_gpu_sweep_full.py tests/test_gpu_bias.py tests/test_gpu_act.py tests/test_presets.py tests/test_gpu_f32x3.py -x -q -k "tf32 or mixed or preset or f32x3" > gpurun_out/ec4_test.txt 2>&1; echo "rc=$?" >> gpurun_out/ec4_test.txt
python scripts/ks_time.py --math tf32 --layout bsf --filter dgt1 --tag ec4 > gpurun_out/ec4_time.jsonl 2>&1
python scripts/time_factors_io.py --cases "1,64,256,16:65536:bsl:bsf;1,64,256,16:65536:bsf:bsf;1,256,64,16:65536:bsf:bsl;1,256,64,16:65536:bsf:bsf" --tag ec4 >> gpurun_out/ec4_time.jsonl 2>&1
python scripts/prof_roles.py "1,64,256,16:65536:bsl:bsf;1,64,64,32:25088:bsf:bsf" > gpurun_out/ec4_roles.txt 2>&1
python scripts/time_models.py --reps 20 --tag ec4 > gpurun_out/ec4_models.jsonl 2>&1
