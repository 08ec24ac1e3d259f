#!/bin/bash
# session 5, last call: the whole GPU suite as the driver runs it, smoke, the default bench line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/s5p_suite.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/s5p_bench_default.json 2> gpurun_out/s5p_bench_default.err
python -c "import json; d=json.load(open('gpurun_out/s5p_bench_default.json')); print('default', d['steps'], d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
