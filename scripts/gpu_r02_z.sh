#!/bin/bash
# session 3 re-entry check: smoke, the GPU suite, the default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_z.log 2>&1; tail -1 gpurun_out/smoke_z.log
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_z.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_z.log
tail -3 gpurun_out/gpu_tests_z.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4_z.json 2> gpurun_out/bench_c4_z.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4_z.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline'].get('assemble_ms_per_step'), d['clocks'])"
