set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_bias.py -x -q > gpurun_out/v2a_pytest.log 2>&1
echo "exit $?" >> gpurun_out/v2a_pytest.log
for V in 1 0; do
  KS_TF32_V2=$V timeout 300 python scripts/ks_time.py --layout bsl --filter all --tag v$V > gpurun_out/v2a_bsl_v$V.jsonl 2>&1
  KS_TF32_V2=$V timeout 300 python scripts/ks_time.py --layout bsf --filter d1 --tag v$V > gpurun_out/v2a_bsf_v$V.jsonl 2>&1
done
