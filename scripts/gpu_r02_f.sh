#!/bin/bash
# j-wavefront one-sweep (kernel 7) vs the TMA two-pass on configs 4 / 1 (+ lag variants); GPU suite
mkdir -p gpurun_out
O=gpurun_out/kw.jsonl
for c in config4 config1; do
  timeout 300 python scripts/sweep_rate.py $c >> $O 2>&1
  CHECK_VS_TMA=1 SUBSURF_KERNEL=kwave timeout 300 python scripts/sweep_rate.py $c >> $O 2>&1
  for v in kw_lag3 kw_lag4 kw_lag6; do
    SUBSURF_B200_LIB=variants/$v.so SUBSURF_KERNEL=kwave timeout 300 python scripts/sweep_rate.py $c >> $O 2>&1
  done
done
SSB_KWAVE_AXIS=0 SUBSURF_B200_LIB=variants/kw_lag4.so SUBSURF_KERNEL=kwave timeout 300 python scripts/sweep_rate.py config1 >> $O 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_f.log
cat $O | cut -c1-400; tail -3 gpurun_out/gpu_tests_f.log
