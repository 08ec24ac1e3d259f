#!/bin/bash
# round-2 evidence run: GPU suite, smoke, config-4 bench (K=20), reference arm, configs 1 / 2 lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_r.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_r.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4_r.json 2> gpurun_out/bench_c4_r.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_c4_r.json 2> gpurun_out/bench_ref_c4_r.err
timeout 600 python bench.py --config config1 --steps 20 --warmup 3 > gpurun_out/bench_c1_r.json 2> gpurun_out/bench_c1_r.err
timeout 600 python bench.py --config config2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_r.json 2> gpurun_out/bench_c2_r.err
tail -2 gpurun_out/gpu_tests_r.log; tail -1 gpurun_out/smoke_r.log
for f in bench_c4_r bench_ref_c4_r bench_c1_r bench_c2_r; do cut -c1-160 gpurun_out/$f.json; done
