mkdir -p gpurun_out/prof
prof() { name=$1; shift;
  env "$@" ncu --set full --clock-control none --import-source on -k regex:ks_tf32 -s 3 -c 1 -o /tmp/$name -f \
    python scripts/ks_time.py --layout bsf --filter "$PAT" --batch $BATCH --reps 1 > gpurun_out/prof/$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/prof/$name.raw.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/prof/$name.sass.csv.gz
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/prof/$name.details.csv 2>&1
}
PAT="1,768,192,2"; BATCH=25088; prof vit_up1 X=1
PAT="1,256,64,16"; BATCH=65536; prof gpt_up1 X=1
PAT="1,256,64,16"; BATCH=65536; prof gpt_up1_j8 KS_BSFJ_J8=1
du -sh gpurun_out/prof
