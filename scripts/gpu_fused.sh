mkdir -p gpurun_out
python scripts/run_chain.py > gpurun_out/fused_${TAG:-a}.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_fused_chain.py -x -q >> gpurun_out/fused_${TAG:-a}.txt 2>&1
