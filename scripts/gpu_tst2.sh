mkdir -p gpurun_out
python -m pytest tests/test_gpu_tf32.py tests/test_gpu_mixed.py tests/test_gpu_sweep_full.py tests/test_gpu_bias.py tests/test_gpu_act.py -x -q -k "tf32 or mixed" > gpurun_out/tst2_test.txt 2>&1; echo "rc=$?" >> gpurun_out/tst2_test.txt
C="1,96,96,16:25088:bsf:bsf;1,96,96,32:25088:bsf:bsf;1,96,96,48:25088:bsf:bsf;1,96,96,64:25088:bsf:bsf;1,96,96,24:25088:bsf:bsf;1,128,128,16:25088:bsf:bsf;1,128,128,24:25088:bsf:bsf;1,128,128,32:25088:bsf:bsf;1,128,128,48:25088:bsf:bsf;1,128,128,64:25088:bsf:bsf;2,96,96,16:25088:bsf:bsf;2,128,128,16:25088:bsf:bsf;3,128,128,16:25088:bsf:bsf;4,96,96,16:25088:bsf:bsf;1,256,64,16:65536:bsf:bsl;1,256,64,16:65536:bsf:bsf"
for k in 0 8; do python scripts/time_factors_io.py --cases "$C" --knobs $k --tag k$k >> gpurun_out/tst2_j8.jsonl 2>&1; done
KS_TF32_TMASTORE=0 python scripts/time_factors_io.py --cases "$C" --knobs 8 --tag k8notst >> gpurun_out/tst2_j8.jsonl 2>&1
