#!/bin/bash
# column assembly kernel: parity, rate vs the tile kernel, ncu
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -s -k "certified or tile_assembly or assemble or segment" > gpurun_out/col_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/col_tests.log
grep -E "no-margin|passed|failed|rc=|Error|error" gpurun_out/col_tests.log | head -20
O=gpurun_out/asm_col.jsonl
for rep in 1 2; do
for c in config1 config4; do
  for v in 1 0; do
    SSB_ASM_COL=$v timeout 300 python scripts/asm_rate.py $c | sed "s/\"config\"/\"col\": $v, \"config\"/" >> $O 2>&1
  done
done
done
cut -c1-150 $O
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:assemble_col_kernel" -s 2 -c 1 \
    -o gpurun_out/asm_col_c1 -f python scripts/asm_rate.py config1 > gpurun_out/asm_col_c1.log 2>&1
tail -1 gpurun_out/asm_col_c1.log
