#!/bin/bash
# whole-row items (R = 2 rows of 128 slots) vs 2D-tiled items (8 rows x 32 slots) on config 4 under the power cap
mkdir -p gpurun_out
O=gpurun_out/power_tile2d.jsonl
for rep in 1 2; do
  for k in tma tma2d; do
    SUBSURF_KERNEL=$k timeout 300 python scripts/power_probe.py config4 >> $O 2>&1
  done
done
cat $O
