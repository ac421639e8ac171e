# FFMA split-rows tiles for underfilled launches (a = d = 1): parity + A/B timing
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep_full.py tests/test_gpu_cliffs.py tests/test_gpu_bias.py tests/test_gpu_act.py -x -q -k "not tf32 and not half and not f32x3" > gpurun_out/splitm_test.txt 2>&1
echo "rc=$?" >> gpurun_out/splitm_test.txt
for m in 0 1; do for lay in bsf bsl; do
  KS_FFMA_SPLITM=$m python scripts/ks_time.py --math fp32 --layout $lay --filter "1,128,128,1;1,64,64,1;1,96,96,1;1,48,48,1;1,128,128,2" --tag splitm$m >> gpurun_out/splitm_time.jsonl 2>&1
done; done
python scripts/ks_time.py --math fp32 --layout bsf --batch 1024 --filter "1,128,128,1;1,64,64,1" --tag small >> gpurun_out/splitm_time.jsonl 2>&1
