mkdir -p gpurun_out
C="1,64,256,16:65536:bsl:bsf;1,256,64,16:65536:bsf:bsl;64,64,64,1:65536:bsf:bsl;64,64,64,1:65536:bsl:bsf;1,768,192,2:25088:bsf:bsf;1,128,128,3:25088:bsf:bsf;1,64,256,16:65536:bsf:bsf"
for dbg in 0 1 2 3; do
  KS_TF32_DEBUG=$dbg python scripts/time_factors_io.py --cases "$C" --tag dbg$dbg >> gpurun_out/dbg_io.jsonl 2>&1
done
