mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_v2.log 2>&1; echo "pytest exit $?" >> gpurun_out/r02_pytest_gpu_v2.log
timeout 900 python bench.py > gpurun_out/r02_bench_v1.json 2> gpurun_out/r02_bench_v1.err; echo "bench exit $?" >> gpurun_out/r02_bench_v1.err
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r02_smoke.txt 2>&1
