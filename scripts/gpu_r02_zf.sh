#!/bin/bash
# certified gradients in the general tile kernel: GPU suite, bench config 4 and config 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests_f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_f.log
tail -3 gpurun_out/gpu_tests_f.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4_f.json 2> gpurun_out/bench_c4_f.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4_f.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline'].get('assemble_ms_per_step'), d['clocks'])"
timeout 900 python bench.py --config config1 --steps 20 --warmup 3 > gpurun_out/bench_c1_f.json 2> gpurun_out/bench_c1_f.err
python -c "import json; d=json.load(open('gpurun_out/bench_c1_f.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline'].get('assemble_ms_per_step'), d['clocks'])"
