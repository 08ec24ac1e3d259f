#!/bin/bash
# round 2, second GPU pass: full GPU suite, assembly A/B (tile vs old kernel), ncu of the tile kernel
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_b.log
for c in config1 config4; do
  timeout 300 python scripts/asm_rate.py $c >> gpurun_out/asm_ab.jsonl 2>&1
  SSB_ASM_TILE=0 timeout 300 python scripts/asm_rate.py $c | sed 's/"config"/"old_kernel": 1, "config"/' >> gpurun_out/asm_ab.jsonl 2>&1
done
if timeout 300 python scripts/asm_rate.py config1 > /dev/null 2>&1; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:assemble_tile_kernel -s 2 -c 1 \
     -o gpurun_out/asm_tile_c1 -f python scripts/asm_rate.py config1 > gpurun_out/asm_tile_c1.log 2>&1
  SSB_ASM_TILE=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:assemble_kernel -s 4 -c 1 \
     -o gpurun_out/asm_old_c1 -f python scripts/asm_rate.py config1 > gpurun_out/asm_old_c1.log 2>&1
fi
tail -5 gpurun_out/gpu_tests_b.log; cat gpurun_out/asm_ab.jsonl
