#!/bin/bash
# 32 planes per item: GPU suite (pins: iteration counts and u bits), bench config 4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_p32.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_p32.log
tail -3 gpurun_out/gpu_tests_p32.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4_p32.json 2> gpurun_out/bench_c4_p32.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4_p32.json')); print('c4', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
