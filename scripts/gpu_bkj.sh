mkdir -p gpurun_out
C="1,768,192,2;1,128,128,3;1,128,128,4;16,128,128,4;4,96,96,4;1,128,128,16;2,64,64,16;1,64,256,16;1,256,64,16;1,96,96,6;6,64,64,4"
O=gpurun_out/bkj.jsonl; : > $O
python scripts/ks_time.py --layout bsf --math tf32 --reps 10 --filter "$C" --tag base >> $O 2>&1
KS_BSFJ_BKJ8=1 python scripts/ks_time.py --layout bsf --math tf32 --reps 10 --filter "$C" --tag bkj8 >> $O 2>&1
KS_BSFJ_BKJ8=1 timeout 600 python -m pytest tests/test_gpu_tf32.py -x -q -k "bsf" > gpurun_out/bkj_pytest.log 2>&1; echo "exit $?" >> gpurun_out/bkj_pytest.log
