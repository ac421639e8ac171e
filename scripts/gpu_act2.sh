mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_act.py tests/test_gpu_half.py -q > gpurun_out/act2_pytest.log 2>&1; echo "exit $?" >> gpurun_out/act2_pytest.log
for i in 1 2; do python bench.py --steps 100 --warmup 5 --no-sweep --no-models --no-cpu-baseline --no-e2e --no-baselines --no-verify > gpurun_out/act2_bench_$i.json 2>/dev/null; done
python - > gpurun_out/act2_sweep_bf16.json 2>&1 <<'PY'
import sys, json, torch
sys.path.insert(0, '.')
import bench_sweep
r = bench_sweep.run_sweep(torch.device('cuda:0'), reps=7, math='bf16', check=False)
print(json.dumps({k: v for k, v in r.items() if 'median' in k}))
PY
