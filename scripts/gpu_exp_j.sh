mkdir -p gpurun_out
C="1,768,192,2:25088:bsl:bsf;1,768,192,2:25088:bsf:bsf;1,768,192,2:25088:bsf:bsl;1,128,128,3:25088:bsl:bsf;1,128,128,3:25088:bsf:bsf;1,64,256,16:65536:bsl:bsf;1,64,256,16:65536:bsf:bsf;1,256,64,16:65536:bsf:bsl;1,256,64,16:65536:bsf:bsf;1,128,128,4:25088:bsf:bsf;1,128,128,4:25088:bsl:bsf;1,128,128,4:25088:bsf:bsl;1,128,128,4:25088:bsl:bsl;1,128,128,16:25088:bsf:bsf;1,128,128,16:25088:bsl:bsl"
O=gpurun_out/exp_j_${TAG:-a}.jsonl
: > $O
python scripts/time_factors_io.py --cases "$C" --tag base >> $O 2>&1
KS_TF32_DEBUG=1 python scripts/time_factors_io.py --cases "$C" --tag nostore >> $O 2>&1
KS_TF32_DEBUG=2 python scripts/time_factors_io.py --cases "$C" --tag nostgread >> $O 2>&1
KS_TF32_DEBUG=3 python scripts/time_factors_io.py --cases "$C" --tag neither >> $O 2>&1
