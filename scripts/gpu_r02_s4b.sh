#!/bin/bash
# session 4: scaled face gradients in the edge tile kernel -- GPU suite, prepare phases on config 4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tile_face or preprocess" 2>&1 | tail -3
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_s4b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_s4b.log
tail -2 gpurun_out/gpu_tests_s4b.log
for v in 1 0 1 0; do
  echo "SSB_EDGE_SCALED=$v"
  SSB_EDGE_SCALED=$v SSB_TIMING=1 timeout 600 python scripts/prep_twice.py config4 2>&1 | grep -E "face_coef|prepare"
done
