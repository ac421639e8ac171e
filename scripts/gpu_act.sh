mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_act.py tests/test_gpu_bias.py tests/test_gpu_mixed.py tests/test_gpu_fused_chain.py -q > gpurun_out/act_pytest.log 2>&1; echo "exit $?" >> gpurun_out/act_pytest.log
