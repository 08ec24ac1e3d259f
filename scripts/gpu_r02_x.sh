#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4_x.json 2> gpurun_out/bench_c4_x.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4_x.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['assemble_ms_per_step'], d['clocks'])"
