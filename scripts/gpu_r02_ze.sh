#!/bin/bash
# certified kernel with ping-pong G registers; 1 CTA/SM variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -s -k "certified or tile_assembly" > gpurun_out/cert_tests_e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/cert_tests_e.log
grep -E "no-margin|passed|failed|rc=" gpurun_out/cert_tests_e.log
O=gpurun_out/asm_var_e.jsonl
for c in config1 config4; do
  for v in "1 base" "0 base" "1 minb1" "0 minb1" "1 minb1st3"; do
    set -- $v
    if [ $2 = base ]; then L=; else L=variants/$2.so; fi
    SUBSURF_B200_LIB=$L SSB_ASM_CERTK=$1 timeout 300 python scripts/asm_rate.py $c | sed "s/\"config\"/\"certk\": $1, \"config\"/" >> $O 2>&1
  done
done
cut -c1-150 $O
