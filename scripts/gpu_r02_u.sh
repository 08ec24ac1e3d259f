#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_bench_dist.py -m gpu -q 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_u.json 2> gpurun_out/bench_c4_u.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4_u.json')); print(d['value'], d['e2e'], d['roofline']['frac'], d['clocks'])"
