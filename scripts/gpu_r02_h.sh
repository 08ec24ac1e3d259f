#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_dist.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/gpu_tests_h.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_h.log
tail -15 gpurun_out/gpu_tests_h.log
