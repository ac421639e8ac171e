mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_v3.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_pytest_gpu_v3.log
timeout 300 python scripts/time_small_b.py > gpurun_out/small_b.jsonl 2>&1
