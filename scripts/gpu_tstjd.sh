mkdir -p gpurun_out
python -m pytest tests/test_gpu_tf32.py tests/test_gpu_mixed.py tests/test_gpu_bias.py tests/test_gpu_act.py tests/test_gpu_sweep_full.py -x -q -k "tf32 or mixed" > gpurun_out/tstjd_test.txt 2>&1; echo "rc=$?" >> gpurun_out/tstjd_test.txt
for g in 1 3; do KS_TF32_MAXGRID=$g python tests/multitile_check.py >> gpurun_out/tstjd_test.txt 2>&1; echo "mt rc=$?" >> gpurun_out/tstjd_test.txt; done
P="1,48,48,4;2,48,48,4;4,64,64,4;8,96,96,4;16,128,128,4;1,128,128,4;3,96,96,4;6,64,64,4;12,48,48,4;1,64,64,8;1,128,128,8;1,96,96,8;1,48,48,8;1,128,128,2;1,96,96,2;1,64,64,2;2,128,128,2;1,128,128,6;1,96,96,3"
for t in 0 1; do KS_TF32_TMASTORE=$t python scripts/ks_time.py --math tf32 --layout bsf --filter "$P" --tag t$t >> gpurun_out/tstjd_time.jsonl 2>&1; done
bash scripts/prof_r03.sh > gpurun_out/prof_r03.log 2>&1
