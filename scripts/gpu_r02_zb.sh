#!/bin/bash
# ncu --set full of the certified assembly tile kernel (config 1, 3rd launch)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:assemble_tile_kernel" -s 2 -c 1 \
    -o gpurun_out/asm_cert_c1 -f python scripts/asm_rate.py config1 > gpurun_out/asm_cert_c1.log 2>&1
tail -3 gpurun_out/asm_cert_c1.log
