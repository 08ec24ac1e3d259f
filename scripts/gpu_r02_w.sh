#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_w.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_w.log
O=gpurun_out/asm_w.jsonl
for c in config1 config4; do
  timeout 300 python scripts/asm_rate.py $c >> $O 2>&1
  SSB_ASM_NR1=0 timeout 300 python scripts/asm_rate.py $c | sed 's/"config"/"nr1": 0, "config"/' >> $O 2>&1
  SSB_ASM_SCALED=0 timeout 300 python scripts/asm_rate.py $c | sed 's/"config"/"scaled": 0, "config"/' >> $O 2>&1
  SSB_ASM_NR1=0 SSB_ASM_SCALED=0 timeout 300 python scripts/asm_rate.py $c | sed 's/"config"/"nr1": 0, "scaled": 0, "config"/' >> $O 2>&1
done
tail -3 gpurun_out/gpu_tests_w.log; cut -c1-130 $O
