#!/bin/bash
# session 5: config 2 pinned for all 30 steps -- the pin tests
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pins.py -m gpu -q -x --durations=6 2>&1 | tail -12
