#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_e.log
tail -5 gpurun_out/gpu_tests_e.log
