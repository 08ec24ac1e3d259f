#!/bin/bash
# assembly: G loads issued at the top of the plane (volatile) vs sunk to the tail
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "certified or tile_assembly or assemble" > gpurun_out/gearly_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gearly_tests.log
tail -2 gpurun_out/gearly_tests.log
O=gpurun_out/asm_gearly.jsonl
for rep in 1 2; do
for c in config1 config4; do
  for v in base glate; do
    if [ $v = base ]; then L=; else L=variants/$v.so; fi
    SUBSURF_B200_LIB=$L timeout 300 python scripts/asm_rate.py $c 2>&1 | tail -1 | sed "s/\"config\"/\"var\": \"$v\", \"config\"/" >> $O
  done
done
done
cut -c1-120 $O
