mkdir -p gpurun_out
P="1,128,128,64;16,128,128,4;1,64,64,64;1,128,128,12;4,64,64,16;1,48,48,64;1,96,96,24"
run() { tag=$1; shift; env "$@" timeout 120 python scripts/ks_time.py --layout bsl --filter "$P" --tag $tag >> gpurun_out/v2b.jsonl 2>&1; }
rm -f gpurun_out/v2b.jsonl
run v1 KS_TF32_V2=0
run o0 KS_V2_ORDER=0
run o1 KS_V2_ORDER=1
run o1k2 KS_V2_ORDER=1 KS_V2_NKB=2
run o0s4 KS_V2_ORDER=0 KS_V2_SMAX=4
run o1k1 KS_V2_ORDER=1 KS_V2_NKB=1
for tag in v1 o1; do
  KS_TF32_V2=$([ $tag = v1 ] && echo 0 || echo 1) KS_V2_ORDER=1 timeout 120 python scripts/ks_time.py --layout bsf --filter "1,128,128,1;1,64,64,1;64,64,64,1;6,64,256,1;16,128,128,1" --tag bsf_$tag >> gpurun_out/v2b.jsonl 2>&1
done
KS_V2_ORDER=0 timeout 120 python scripts/ks_time.py --layout bsf --filter "1,128,128,1;1,64,64,1;64,64,64,1;6,64,256,1;16,128,128,1" --tag bsf_o0 >> gpurun_out/v2b.jsonl 2>&1
