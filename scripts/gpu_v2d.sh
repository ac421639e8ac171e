mkdir -p gpurun_out
P="1,128,128,64;16,128,128,4;1,64,64,64;1,128,128,12;4,64,64,16;1,48,48,64;1,96,96,24"
run() { tag=$1; lay=$2; pp=$3; shift; shift; shift; env "$@" timeout 120 python scripts/ks_time.py --layout $lay --filter "$pp" --tag $tag >> gpurun_out/v2d.jsonl 2>&1; }
rm -f gpurun_out/v2d.jsonl
run v1 bsl "$P" KS_TF32_V2=0
run o0 bsl "$P" KS_V2_ORDER=0
run o4 bsl "$P" KS_V2_ORDER=4
run o5 bsl "$P" KS_V2_ORDER=5
Q="1,128,128,1;1,64,64,1;64,64,64,1;6,64,256,1;16,128,128,1;6,64,64,1"
run v1 bsf "$Q" KS_TF32_V2=0
run o0 bsf "$Q" KS_V2_ORDER=0
run o0k2 bsf "$Q" KS_V2_ORDER=0 KS_V2_NKB=2
run o1 bsf "$Q" KS_V2_ORDER=1
run o1k2 bsf "$Q" KS_V2_ORDER=1 KS_V2_NKB=2
run o0nf bsf "$Q" KS_V2_ORDER=0 KS_V2_FILL=0
# correctness of the 5-D canonical layout
KS_V2_ORDER=4 timeout 300 python -m pytest tests/test_gpu_tf32.py -x -q -k "matches_oracle or integer" > gpurun_out/v2d_o4_pytest.log 2>&1
echo "exit $?" >> gpurun_out/v2d_o4_pytest.log
