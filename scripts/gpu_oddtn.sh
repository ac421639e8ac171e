mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep_full.py tests/test_gpu_cliffs.py tests/test_gpu_bias.py tests/test_gpu_act.py -x -q -k "not tf32 and not half and not f32x3" > gpurun_out/oddtn_test.txt 2>&1; echo "rc=$?" >> gpurun_out/oddtn_test.txt
for g in 1 3 7; do KS_TF32_MAXGRID=$g KS_MULTITILE_MATH=fp32 python tests/multitile_check.py >> gpurun_out/oddtn_test.txt 2>&1; echo "mt rc=$?" >> gpurun_out/oddtn_test.txt; done
P="1,96,96,1;1,48,48,1;1,128,128,1;1,64,64,1;2,96,96,1;2,48,48,1"
for m in 0 1 0 1; do for lay in bsf bsl; do
  KS_FFMA_SPLITM=$m python scripts/ks_time.py --math fp32 --layout $lay --filter "$P" --tag m$m >> gpurun_out/oddtn_time.jsonl 2>&1
done; done
