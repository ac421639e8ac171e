#!/bin/bash
# TF32 BSF J-gather iteration: parity tests of the tcgen05 families, then the TF32 sweep and model lines.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_f32x3.py tests/test_gpu_bias.py -q -x > gpurun_out/pytest_tf32j.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_tf32j.log
timeout 900 python bench_sweep.py tf32 > gpurun_out/sweep_tf32.json 2> gpurun_out/sweep_tf32.err
MATHS="tf32 f32x3" STEPS=30 bash scripts/bench_models.sh
