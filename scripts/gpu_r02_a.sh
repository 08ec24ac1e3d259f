#!/bin/bash
# round 2, first GPU pass: host facts, the GPU suite, config-4 bench (both arms)
mkdir -p gpurun_out
{ nproc; free -g; lscpu | grep -i "model name"; nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv; } > gpurun_out/host.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?" >> gpurun_out/bench_c4.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_c4.json 2> gpurun_out/bench_ref_c4.err; echo "ref rc=$?" >> gpurun_out/bench_ref_c4.err
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/bench_c4.json | cut -c1-600
