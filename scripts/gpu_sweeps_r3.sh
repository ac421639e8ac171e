mkdir -p gpurun_out
python -m pytest tests/test_gpu_fused_chain.py -x -q > gpurun_out/fused_pf1_test.txt 2>&1; echo "rc=$?" >> gpurun_out/fused_pf1_test.txt
python scripts/run_chain.py > gpurun_out/fused_pf1_time.txt 2>&1
python scripts/sweep_rows.py tf32 > gpurun_out/sweep_tf32.log 2>&1
python scripts/sweep_rows.py fp32 > gpurun_out/sweep_fp32.log 2>&1
