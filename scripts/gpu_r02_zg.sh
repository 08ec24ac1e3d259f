#!/bin/bash
# config-4 steady-state red pass, ncu --set full with source counters
mkdir -p gpurun_out
bash scripts/ncu_pass.sh config4 sor_c4_red_g
tail -2 gpurun_out/sor_c4_red_g.log
