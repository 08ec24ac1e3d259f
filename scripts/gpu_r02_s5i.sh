#!/bin/bash
# session 5: what leaving CTA slots free costs the persistent SOR pass (room for NCCL's send/recv kernels on a
# distributed run): SSB_GRID_SHORT = 0 / 4 / 8 / 16 / 32 / 64 of the 296 slots, power-capped 3000-sweep loops
mkdir -p gpurun_out
for cfg in config4 config1; do
  for gs in 0 8 0 16 32 4 64 0; do
    SSB_GRID_SHORT=$gs timeout 300 python scripts/power_probe.py $cfg 2>/dev/null | tail -1 | sed "s/^/{\"grid_short\": $gs, \"r\": /; s/$/}/" | tee -a gpurun_out/s5i_grid_short.jsonl
  done
done
