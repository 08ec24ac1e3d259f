#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_i.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4_i.json 2> gpurun_out/bench_c4_i.err
tail -4 gpurun_out/gpu_tests_i.log; cut -c1-300 gpurun_out/bench_c4_i.json
