mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_mixed.py -x -q > gpurun_out/mixed_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/mixed_pytest.log
