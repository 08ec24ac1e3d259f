mkdir -p gpurun_out
timeout 1200 python scripts/track_bench.py config2 | tee gpurun_out/track_config2.json
