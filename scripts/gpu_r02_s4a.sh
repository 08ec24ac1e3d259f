#!/bin/bash
# session 4: validate the restored tree (smoke, GPU suite, config-4 bench line)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_s4a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_s4a.log
tail -2 gpurun_out/gpu_tests_s4a.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4_s4a.json 2> gpurun_out/bench_c4_s4a.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4_s4a.json')); print('c4', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline'].get('assemble_ms_per_step'), d['clocks'])"
