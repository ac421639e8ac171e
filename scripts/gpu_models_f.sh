mkdir -p gpurun_out; rm -f gpurun_out/models_f.jsonl
V="1,768,192,2;6,64,64,1;1,128,128,3;6,64,256,1"
G="1,64,256,16;64,64,64,1;1,256,64,16"
run() { tag=$1; shift; env "$@" timeout 300 python scripts/ks_time.py --layout bsf --filter "$V" --batch 25088 --tag $tag >> gpurun_out/models_f.jsonl 2>&1;
                       env "$@" timeout 300 python scripts/ks_time.py --layout bsf --filter "$G" --batch 65536 --tag $tag >> gpurun_out/models_f.jsonl 2>&1; }
run base KS_TF32_V2=0
run j8 KS_BSFJ_J8=1
run v2 KS_TF32_V2=1 KS_V2_ORDER=0
run v2k2 KS_TF32_V2=1 KS_V2_NKB=2

for P in "1,768,192,2;6,64,64,1;1,128,128,3;6,64,256,1"; do timeout 300 python scripts/ks_time.py --math fp32 --layout bsf --filter "$P" --batch 25088 --tag fp32 >> gpurun_out/models_f.jsonl 2>&1; done
timeout 300 python scripts/ks_time.py --math fp32 --layout bsf --filter "1,64,256,16;64,64,64,1;1,256,64,16" --batch 65536 --tag fp32 >> gpurun_out/models_f.jsonl 2>&1
