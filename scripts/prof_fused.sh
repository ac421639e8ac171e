mkdir -p gpurun_out/prof_fused
name=fused
ncu --set full --clock-control none --import-source on -k regex:ks_chain_fused -s 2 -c 1 -o gpurun_out/prof_fused/$name -f \
    python scripts/run_chain.py > gpurun_out/prof_fused/$name.log 2>&1
ncu -i gpurun_out/prof_fused/$name.ncu-rep --page raw --csv > gpurun_out/prof_fused/$name.raw.csv 2>&1
ncu -i gpurun_out/prof_fused/$name.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/prof_fused/$name.sass.csv.gz
rm -f gpurun_out/prof_fused/$name.ncu-rep
