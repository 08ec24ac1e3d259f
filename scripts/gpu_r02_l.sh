#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_l.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_l.log
O=gpurun_out/power_l.jsonl
timeout 300 python scripts/power_probe.py config4 >> $O 2>&1
SUBSURF_B200_LIB=variants/nores.so timeout 300 python scripts/power_probe.py config4 >> $O 2>&1
timeout 300 python scripts/power_probe.py config4 >> $O 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4_l.json 2> gpurun_out/bench_c4_l.err
tail -3 gpurun_out/gpu_tests_l.log; cat $O; cut -c1-200 gpurun_out/bench_c4_l.json
