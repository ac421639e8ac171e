#!/bin/bash
# One gpurun pass: build, smoke, GPU tests, bench (+ sweep), ncu launch list + one full capture.
#   STAGES="smoke tests bench sweep ncu" (default all)
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
STAGES="${STAGES:-smoke tests bench sweep ncu}"
nvidia-smi > gpurun_out/nvidia_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [[ $STAGES == *smoke* ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
fi
if [[ $STAGES == *tests* ]]; then
  timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
if [[ $STAGES == *bench* ]]; then
  timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
fi
if [[ $STAGES == *sweep* ]]; then
  for m in ${SWEEP_MODES:-fp32 tf32}; do
    timeout 900 python bench_sweep.py $m > gpurun_out/sweep_$m.json 2> gpurun_out/sweep_$m.err
  done
fi
if [[ $STAGES == *ncu* ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-sweep --no-verify --no-baselines \
      > gpurun_out/ncu_launch_bench.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-ks_stream} -s ${NCU_SKIP:-12} -c ${NCU_COUNT:-3} \
      -o gpurun_out/prof_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-sweep --no-verify --no-baselines ${NCU_BENCH_ARGS} \
      > gpurun_out/ncu_full.log 2>&1
fi
ls -la gpurun_out
