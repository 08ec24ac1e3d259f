#!/bin/bash
# step_host_async: tests, bench config 4 (e2e through the chained async call)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_slabs.py -m gpu -q -x -k "step_host" > gpurun_out/async_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/async_tests.log
tail -3 gpurun_out/async_tests.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4_q.json 2> gpurun_out/bench_c4_q.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4_q.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline'].get('assemble_ms_per_step'), d['clocks'])"
tail -3 gpurun_out/bench_c4_q.err
