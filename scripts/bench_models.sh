#!/bin/bash
# configs[3]/[4] bench lines: ViT-S/16 and GPT-2 medium KSLinear chains, FP32 / TF32 / 3xTF32, BSF,
# with the bmm+permute and dense cuBLAS baselines of the same chain.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for wl in ${WORKLOADS:-vit_up vit_down gpt2_down gpt2_up}; do
  for m in ${MATHS:-fp32 tf32 f32x3}; do
    timeout 300 python bench.py --workload $wl --math $m --steps ${STEPS:-50} --warmup 5 --no-sweep --no-cpu-baseline \
        > gpurun_out/bench_${wl}_${m}.json 2> gpurun_out/bench_${wl}_${m}.err
  done
done
