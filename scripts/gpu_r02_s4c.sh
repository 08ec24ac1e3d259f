#!/bin/bash
# session 4: edge tile kernel -- 1 stage x 2 CTAs/SM vs 2 stages x 1 CTA/SM, scaled vs exact gradients
mkdir -p gpurun_out
for st in 1 2; do
  SSB_EDGE_STAGES=$st timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "tile_face or preprocess" 2>&1 | tail -1
done
for rep in 1 2; do
for st in 1 2; do
for v in 1 0; do
  echo "STAGES=$st SCALED=$v: $(SSB_EDGE_STAGES=$st SSB_EDGE_SCALED=$v SSB_TIMING=1 timeout 600 python scripts/prep_twice.py config4 2>&1 | grep -E "face_coef" | tail -1)"
done; done; done
