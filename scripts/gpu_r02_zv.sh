#!/bin/bash
# host-transfer chunks 16 vs 8: tests, bench e2e
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slabs.py -m gpu -q -x -k "step_host" > gpurun_out/hc_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/hc_tests.log
tail -2 gpurun_out/hc_tests.log
for v in base hc8 base hc8; do
  if [ $v = base ]; then L=; else L=variants/$v.so; fi
  SUBSURF_B200_LIB=$L timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_hc_$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/bench_hc_$v.json')); print('$v', d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks']['sm_mhz'])"
done
