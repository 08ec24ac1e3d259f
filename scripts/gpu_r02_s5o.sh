#!/bin/bash
# session 5: ncu --set full of the assembly tile kernel and the one-off edge tile kernel on config 4
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:assemble_tile_kernel -s 1 -c 1 \
    -o gpurun_out/s5_asm_c4 -f python scripts/asm_rate.py config4 > gpurun_out/s5_asm_c4.log 2>&1
tail -2 gpurun_out/s5_asm_c4.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:edge_tile_kernel -c 1 \
    -o gpurun_out/s5_edge_c4 -f python scripts/asm_rate.py config4 > gpurun_out/s5_edge_c4.log 2>&1
tail -2 gpurun_out/s5_edge_c4.log
