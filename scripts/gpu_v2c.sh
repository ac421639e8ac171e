mkdir -p gpurun_out
P="1,128,128,64;16,128,128,4;1,64,64,64;1,128,128,12;4,64,64,16;1,48,48,64;1,96,96,24"
run() { tag=$1; shift; env "$@" timeout 120 python scripts/ks_time.py --layout bsl --filter "$P" --tag $tag >> gpurun_out/v2c.jsonl 2>&1; }
rm -f gpurun_out/v2c.jsonl
run v1 KS_TF32_V2=0
run o0 KS_V2_ORDER=0
run o2 KS_V2_ORDER=2
run o3 KS_V2_ORDER=3
