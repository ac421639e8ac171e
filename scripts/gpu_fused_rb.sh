# register-blocked fused chain: parity + A/B timing + ncu of the fused kernel
mkdir -p gpurun_out
python -m pytest tests/test_gpu_fused_chain.py -x -q > gpurun_out/fused_rb_test.txt 2>&1
echo "test rc=$?" >> gpurun_out/fused_rb_test.txt
for rb in 0 1; do
  KS_FUSED_RB=$rb python scripts/run_chain.py >> gpurun_out/fused_rb_time.txt 2>&1
  KS_FUSED_RB=$rb python scripts/run_chain.py 11 8192 >> gpurun_out/fused_rb_time.txt 2>&1
done
sed -i 's/^/rb? /' /dev/null
name=fused_rb
ncu --set full --clock-control none --import-source on -k regex:ks_chain_fused -s 2 -c 1 -o gpurun_out/$name -f \
    python scripts/run_chain.py > gpurun_out/$name.log 2>&1
ncu -i gpurun_out/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>&1
ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/$name.sass.csv.gz
rm -f gpurun_out/$name.ncu-rep
