# ncu --set full captures of the round-2-late kernels (MNJ, J = 8 TMA-store, d = 1 TMA-store, fused chain)
mkdir -p gpurun_out/prof_r03
prof() { name=$1; cs=$2; shift 2;
  env "$@" ncu --set full --clock-control none --import-source on -k regex:ks_ -s 3 -c 1 -o gpurun_out/prof_r03/$name -f \
    python scripts/time_factors_io.py --cases "$cs" --reps 1 > gpurun_out/prof_r03/$name.log 2>&1
  ncu -i gpurun_out/prof_r03/$name.ncu-rep --page raw --csv > gpurun_out/prof_r03/$name.raw.csv 2>&1
  ncu -i gpurun_out/prof_r03/$name.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/prof_r03/$name.sass.csv.gz
  rm -f gpurun_out/prof_r03/$name.ncu-rep
}
prof mnj_gpt2down2 "1,64,256,16:65536:bsl:bsf"
prof tst_j8 "1,48,48,64:25088:bsf:bsf"
prof tstd_d1 "64,64,64,1:65536:bsl:bsf"
name=fused
ncu --set full --clock-control none --import-source on -k regex:ks_chain_fused -s 2 -c 1 -o gpurun_out/prof_r03/$name -f \
    python scripts/run_chain.py > gpurun_out/prof_r03/$name.log 2>&1
ncu -i gpurun_out/prof_r03/$name.ncu-rep --page raw --csv > gpurun_out/prof_r03/$name.raw.csv 2>&1
rm -f gpurun_out/prof_r03/$name.ncu-rep
du -sh gpurun_out/prof_r03
