#!/bin/bash
# assembly tail (one-compare midpoint test, float-exponent range) + wait-hint / stage variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -s -k "certified or tile_assembly or assemble or segment" > gpurun_out/cert_tests_c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/cert_tests_c.log
grep -E "no-margin|passed|failed|rc=" gpurun_out/cert_tests_c.log
O=gpurun_out/asm_var_c.jsonl
for rep in 1 2; do
for c in config1 config4; do
  for v in base susp1k susp10k st3; do
    if [ $v = base ]; then L=; else L=variants/$v.so; fi
    SUBSURF_B200_LIB=$L timeout 300 python scripts/asm_rate.py $c >> $O 2>&1
  done
done
done
cut -c1-150 $O
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:assemble_tile_kernel" -s 2 -c 1 \
    -o gpurun_out/asm_cert2_c1 -f python scripts/asm_rate.py config1 > gpurun_out/asm_cert2_c1.log 2>&1
tail -1 gpurun_out/asm_cert2_c1.log
