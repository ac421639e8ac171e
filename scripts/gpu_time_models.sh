mkdir -p gpurun_out
timeout 600 python scripts/time_models.py --tag ${TAG:-m} > gpurun_out/time_models_${TAG:-m}.jsonl 2> gpurun_out/time_models_${TAG:-m}.err
