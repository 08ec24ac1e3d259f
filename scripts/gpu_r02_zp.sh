#!/bin/bash
# column assembly: ring depths after the step-counter fix
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -s -k "certified or tile_assembly or assemble or segment" > gpurun_out/col_tests_p.log 2>&1; echo "pytest rc=$?" >> gpurun_out/col_tests_p.log
grep -E "no-margin|passed|failed|rc=" gpurun_out/col_tests_p.log | head
O=gpurun_out/asm_col_p.jsonl
for c in config1 config4; do
  for v in "0 base" "1 base" "1 nb4g2" "1 nb6g3" "1 nb5g4"; do
    set -- $v
    if [ $2 = base ]; then L=; else L=variants/$2.so; fi
    SUBSURF_B200_LIB=$L SSB_ASM_COL=$1 timeout 300 python scripts/asm_rate.py $c 2>&1 | tail -1 | sed "s/\"config\"/\"col\": \"$1 $2\", \"config\"/" >> $O 2>&1
  done
done
cut -c1-130 $O
