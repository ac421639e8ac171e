mkdir -p gpurun_out; rm -f gpurun_out/dense.jsonl
timeout 600 python -m pytest tests/test_gpu_tf32_dense.py tests/test_gpu_tf32.py tests/test_gpu_bias.py -x -q > gpurun_out/dense_pytest.log 2>&1; echo "exit $?" >> gpurun_out/dense_pytest.log
run() { tag=$1; shift; env "$@" timeout 300 python scripts/ks_time.py --layout bsf --filter dgt1 --tag $tag >> gpurun_out/dense.jsonl 2>&1; }
run off KS_TF32_DENSIFY=0
run on KS_TF32_DENSIFY=2
for m in 0 2; do
  KS_TF32_DENSIFY=$m timeout 300 python scripts/ks_time.py --layout bsf --filter "1,768,192,2;1,128,128,3" --batch 25088 --tag m$m >> gpurun_out/dense_models.jsonl 2>&1
done
