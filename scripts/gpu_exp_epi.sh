mkdir -p gpurun_out
C="1,768,192,2:25088:bsl:bsf;1,768,192,2:25088:bsf:bsf;1,128,128,3:25088:bsf:bsf;1,64,256,16:65536:bsf:bsf;1,256,64,16:65536:bsf:bsf;1,128,128,4:25088:bsf:bsf;1,128,128,16:25088:bsf:bsf;64,64,64,1:25088:bsf:bsf;6,64,256,1:25088:bsf:bsf;16,128,128,1:25088:bsf:bsf;1,128,128,1:25088:bsf:bsf;4,96,96,16:25088:bsf:bsf;12,64,64,4:25088:bsf:bsf;1,96,96,24:25088:bsf:bsf"
O=gpurun_out/exp_epi_${TAG:-a}.jsonl
: > $O
python scripts/time_factors_io.py --cases "$C" --tag base >> $O 2>&1
KS_TF32_DEBUG=4 python scripts/time_factors_io.py --cases "$C" --tag direct >> $O 2>&1
