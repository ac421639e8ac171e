mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r03v5_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r03v5_pytest.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r03v5_smoke.txt 2>&1; echo "smoke exit $?" >> gpurun_out/r03v5_smoke.txt
timeout 900 python bench.py > gpurun_out/r03v5_bench.json 2> gpurun_out/r03v5_bench.err; echo "bench exit $?" >> gpurun_out/r03v5_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r03v5_launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-models > gpurun_out/r03v5_ncu.log 2>&1
