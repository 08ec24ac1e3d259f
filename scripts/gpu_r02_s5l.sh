#!/bin/bash
# session 5: fixed-sweep steps without diagnostics skip the pass that only evaluates the last residual
# (SorState::fixed mode 2): tests, bench config 4, launch list of two timed steps
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_pins.py tests/test_gpu_parity.py tests/test_gpu_dist_host.py tests/test_gpu_bench_dist.py -m gpu -q -x 2>&1 | tail -4
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/s5l_bench_c4.json 2> gpurun_out/s5l_bench_c4.err
python -c "import json; d=json.load(open('gpurun_out/s5l_bench_c4.json')); print('c4', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['gpu_launches'], d['clocks'])"
if timeout 600 python scripts/step_launch_list.py config4 2 > gpurun_out/s5l_sll.log 2>&1; then
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/s5l_launches_step_c4.csv python scripts/step_launch_list.py config4 2 > gpurun_out/s5l_ncu_sll.log 2>&1
fi
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/s5l_bench_c4_b.json 2> gpurun_out/s5l_bench_c4_b.err
python -c "import json; d=json.load(open('gpurun_out/s5l_bench_c4_b.json')); print('c4 again', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
