#!/bin/bash
# strength-reduced SOR producers: GPU suite, power-capped sweep rate vs the previous producers
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_u.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_u.log
tail -2 gpurun_out/gpu_tests_u.log
O=gpurun_out/power_prod.jsonl
for rep in 1 2; do
  for v in base oldprod; do
    if [ $v = base ]; then L=; else L=variants/$v.so; fi
    SUBSURF_B200_LIB=$L timeout 300 python scripts/power_probe.py config4 | sed "s/\"config\"/\"var\": \"$v\", \"config\"/" >> $O 2>&1
  done
done
cut -c1-200 $O
bash scripts/ncu_pass.sh config4 sor_c4_red_u
tail -1 gpurun_out/sor_c4_red_u.log
