#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/asm_n.jsonl
for c in config4 config1; do
for v in "" asm_m3s1 asm_m4s1 asm_m3s2; do
  if [ -z "$v" ]; then timeout 300 python scripts/asm_rate.py $c >> $O 2>&1;
  else SUBSURF_B200_LIB=variants/$v.so timeout 300 python scripts/asm_rate.py $c >> $O 2>&1; fi
done
done
cat $O
