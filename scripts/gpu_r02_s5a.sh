#!/bin/bash
# session 5: re-verification of the restored tree -- full GPU suite, smoke, default bench (config 4)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 | tee gpurun_out/s5a_suite.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2 | tee gpurun_out/s5a_smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/s5a_bench_c4.json 2> gpurun_out/s5a_bench_c4.err
python -c "import json; d=json.load(open('gpurun_out/s5a_bench_c4.json')); print('c4', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline'], d['clocks'], d['cpu_baseline'])"
