#!/bin/bash
mkdir -p gpurun_out
for v in nb4g3 nb4g3gf nb4g2gf nb5g2 base; do
  if [ $v = base ]; then L=; else L=variants/$v.so; fi
  echo "== $v"; SUBSURF_B200_LIB=$L timeout 120 python scripts/asm_rate.py config0 2>&1 | tail -1 | cut -c1-150
done
