mkdir -p gpurun_out; rm -f gpurun_out/j8.jsonl
run() { tag=$1; shift; env "$@" timeout 300 python scripts/ks_time.py --layout bsf --filter dgt1 --tag $tag >> gpurun_out/j8.jsonl 2>&1; }
run j4 KS_BSFJ_J8=0
run j8 KS_BSFJ_J8=1
