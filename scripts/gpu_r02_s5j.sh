#!/bin/bash
# session 5: the short persistent grid (comm_reserve / SSB_GRID_SHORT): bit-identity test, the slab / dist
# suites with the new library, and the whole parity suite under SSB_GRID_SHORT=8
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_pins.py -m gpu -q -x -k "short or config1" 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_dist_host.py tests/test_gpu_bench_dist.py -m gpu -q -x 2>&1 | tail -3
SSB_GRID_SHORT=8 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random_cases.py tests/test_gpu_fullsize.py tests/test_gpu_pins.py -m gpu -q -x 2>&1 | tail -3
