mkdir -p gpurun_out
for b in 8192 4096 2048 1024; do
  python bench.py --steps 50 --warmup 5 --batch $b --no-sweep --no-models --no-baselines --no-cpu-baseline --no-e2e > gpurun_out/strong_$b.json 2> gpurun_out/strong_$b.err
done
