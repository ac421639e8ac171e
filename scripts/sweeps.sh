#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench_sweep.py fp32 > gpurun_out/sweep_fp32.json 2> gpurun_out/sweep_fp32.err
timeout 900 python bench_sweep.py tf32 > gpurun_out/sweep_tf32.json 2> gpurun_out/sweep_tf32.err
timeout 900 python bench_sweep.py perm > gpurun_out/perm_share.json 2> gpurun_out/perm.err
