mkdir -p gpurun_out
timeout 2400 python scripts/autotune.py --out gpurun_out/autotune_fp32_bsf.json --only fp32:bsf --reps 10 > gpurun_out/autotune_fp32_bsf.log 2>&1
echo "exit $?" >> gpurun_out/autotune_fp32_bsf.log
