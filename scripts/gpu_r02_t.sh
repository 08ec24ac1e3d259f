#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/asm_t.jsonl
for r in 1 2; do for c in config1 config4; do
  timeout 300 python scripts/asm_rate.py $c >> $O 2>&1
  SUBSURF_B200_LIB=variants/asm_nol1.so timeout 300 python scripts/asm_rate.py $c >> $O 2>&1
done; done
timeout 900 python -m pytest tests/test_gpu_pins.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
cat $O
