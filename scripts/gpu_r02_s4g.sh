#!/bin/bash
# session 4: step_host_async on distributed ranks -- distributed tests, host-buffer tests, bench dist test
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist_host.py tests/test_gpu_bench_dist.py -m gpu -q -x 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_slabs.py -m gpu -q -x -k "step_host" 2>&1 | tail -2
