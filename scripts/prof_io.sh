# ncu --set full of single ks_matmul_io calls (one capture each); raw metrics + per-CUDA-line source page
mkdir -p gpurun_out/prof_io
prof() { name=$1; cs=$2; shift 2;
  env "$@" ncu --set full --clock-control none --import-source on -k regex:ks_ -s 3 -c 1 -o gpurun_out/prof_io/$name -f \
    python scripts/time_factors_io.py --cases "$cs" --reps 1 > gpurun_out/prof_io/$name.log 2>&1
  ncu -i gpurun_out/prof_io/$name.ncu-rep --page raw --csv > gpurun_out/prof_io/$name.raw.csv 2>&1
  ncu -i gpurun_out/prof_io/$name.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/prof_io/$name.sass.csv.gz
  ncu -i gpurun_out/prof_io/$name.ncu-rep --page details --csv > gpurun_out/prof_io/$name.details.csv 2>&1
  rm -f gpurun_out/prof_io/$name.ncu-rep
}
prof vitup_lf "1,768,192,2:25088:bsl:bsf"
prof gptup1_fl "1,256,64,16:65536:bsf:bsl"
prof a1d4_ll "1,128,128,4:25088:bsl:bsl"
prof a64_ff "64,64,64,1:25088:bsf:bsf"
du -sh gpurun_out/prof_io
