# fused chain: where the next group's load is issued (KS_FUSED_PF_PASS), parity + timing
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fused_chain.py -x -q > gpurun_out/fused_pf_test.txt 2>&1
echo "test rc=$?" >> gpurun_out/fused_pf_test.txt
for pf in -1 0 1 2; do
  echo "pf=$pf" >> gpurun_out/fused_pf_time.txt
  KS_FUSED_PF_PASS=$pf python scripts/run_chain.py >> gpurun_out/fused_pf_time.txt 2>&1
  KS_FUSED_PF_PASS=$pf python scripts/run_chain.py 11 8192 >> gpurun_out/fused_pf_time.txt 2>&1
done
