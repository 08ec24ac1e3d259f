#!/bin/bash
# GPU suite + config-4 bench (e2e through step_host) + config-1 bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_d.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4_d.json 2> gpurun_out/bench_c4_d.err
timeout 600 python bench.py --config config1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1_d.json 2> gpurun_out/bench_c1_d.err
tail -3 gpurun_out/gpu_tests_d.log; cut -c1-400 gpurun_out/bench_c4_d.json; tail -2 gpurun_out/bench_c4_d.err
