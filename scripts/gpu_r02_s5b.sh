#!/bin/bash
# session 5: is the box slow?  bandwidth probes, clocks, then the failing bench-dist test with its output
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,clocks.max.mem,power.draw,temperature.gpu,memory.used,ecc.mode.current,clocks_throttle_reasons.active --format=csv | tee gpurun_out/s5b_smi.txt
nvidia-smi --query-compute-apps=pid,used_memory --format=csv | tee -a gpurun_out/s5b_smi.txt
nproc | tee -a gpurun_out/s5b_smi.txt
timeout 300 python scripts/bw_probe.py 2>&1 | tail -8 | tee gpurun_out/s5b_bw.txt
timeout 300 python scripts/sweep_rate.py config4 2>&1 | tail -6 | tee gpurun_out/s5b_sweep.txt
timeout 900 python -m pytest tests/test_gpu_bench_dist.py -m gpu -q -x 2>&1 | tail -40 | tee gpurun_out/s5b_dist.log
