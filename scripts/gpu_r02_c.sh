#!/bin/bash
# GPU suite + assembly timing (tile kernel with per-warp release + G prefetch) + ncu of it
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_c.log
for c in config1 config4; do
  timeout 300 python scripts/asm_rate.py $c >> gpurun_out/asm_c.jsonl 2>&1
  SSB_ASM_GPREF=0 timeout 300 python scripts/asm_rate.py $c | sed 's/"config"/"gpref": 0, "config"/' >> gpurun_out/asm_c.jsonl 2>&1
done
if timeout 300 python scripts/asm_rate.py config1 > /dev/null 2>&1; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:assemble_tile_kernel -s 2 -c 1 \
     -o gpurun_out/asm_tile2_c1 -f python scripts/asm_rate.py config1 > gpurun_out/asm_tile2_c1.log 2>&1
fi
tail -5 gpurun_out/gpu_tests_c.log; cat gpurun_out/asm_c.jsonl
