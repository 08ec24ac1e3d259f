#!/bin/bash
# ncu --set full of a steady-state config-4 red pass (instruction mix / pipes)
mkdir -p gpurun_out
bash scripts/ncu_pass.sh config4 s4_c4_red
ls -la gpurun_out/s4_c4_red.ncu-rep
tail -3 gpurun_out/s4_c4_red.log
