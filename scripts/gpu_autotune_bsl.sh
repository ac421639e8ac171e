mkdir -p gpurun_out
C="1,48,48,2;1,48,48,4;1,64,64,4;1,96,96,4;1,128,128,4;1,128,128,8;1,64,64,16;1,128,128,16;2,64,64,4;2,128,128,4;3,96,96,4;1,96,96,12;1,128,128,3;1,768,192,2;1,64,256,16;1,256,64,16"
for F in 0 2 4; do KS_BSFJ_FILL=$F python scripts/ks_time.py --layout bsf --math tf32 --reps 10 --filter "$C" --tag fill$F >> gpurun_out/fill.jsonl 2>&1; done
timeout 2400 python scripts/autotune.py --out gpurun_out/autotune_tf32_bsl.json --only tf32:bsl --reps 10 > gpurun_out/autotune_tf32_bsl.log 2>&1
echo "exit $?" >> gpurun_out/autotune_tf32_bsl.log
