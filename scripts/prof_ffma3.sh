mkdir -p gpurun_out/prof_ffma3
prof() { name=$1; cs=$2; shift 2;
  env "$@" ncu --set full --clock-control none --import-source on -k regex:ks_ffma -s 3 -c 1 -o gpurun_out/prof_ffma3/$name -f \
    python scripts/time_factors_io.py --math fp32 --cases "$cs" --reps 1 > gpurun_out/prof_ffma3/$name.log 2>&1
  ncu -i gpurun_out/prof_ffma3/$name.ncu-rep --page raw --csv > gpurun_out/prof_ffma3/$name.raw.csv 2>&1
  ncu -i gpurun_out/prof_ffma3/$name.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/prof_ffma3/$name.sass.csv.gz
  rm -f gpurun_out/prof_ffma3/$name.ncu-rep
}
prof bsl_2_64_16 "2,64,64,16:25088:bsl:bsl"
prof bsl_1_128_12 "1,128,128,12:25088:bsl:bsl"
prof bsf_2_64_16 "2,64,64,16:25088:bsf:bsf"
