#!/bin/bash
# session 5 evidence: the multi-rank tests (retry/watchdog version), bench config 4 (default line) + the
# reference arm, configs 1 / 2, the launch list of exactly the timed steps, the launch list of the
# bench command itself, one steady-state red pass capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bench_dist.py tests/test_gpu_dist_host.py -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/s5_bench_c4.json 2> gpurun_out/s5_bench_c4.err
python -c "import json; d=json.load(open('gpurun_out/s5_bench_c4.json')); print('c4', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['cpu_baseline']['value'])"
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/s5_bench_ref_c4.json 2> gpurun_out/s5_bench_ref_c4.err
python -c "import json; d=json.load(open('gpurun_out/s5_bench_ref_c4.json')); print('ref c4', d['value'], d['ms_per_step'], d['steps'])"
timeout 900 python bench.py --config config1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/s5_bench_c1.json 2> gpurun_out/s5_bench_c1.err
python -c "import json; d=json.load(open('gpurun_out/s5_bench_c1.json')); print('c1', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 python bench.py --config config2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5_bench_c2.json 2> gpurun_out/s5_bench_c2.err
python -c "import json; d=json.load(open('gpurun_out/s5_bench_c2.json')); print('c2', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
if timeout 600 python scripts/step_launch_list.py config4 2 > gpurun_out/s5_sll.log 2>&1; then
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/s5_launches_step_c4.csv python scripts/step_launch_list.py config4 2 > gpurun_out/s5_ncu_sll.log 2>&1
fi
# the bench command itself (loop mode 0: every colour pass its own launch, so ncu lists them)
if timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --loop-mode 0 > gpurun_out/s5_bench_lm0.json 2> gpurun_out/s5_bench_lm0.err; then
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/s5_launches_bench_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --loop-mode 0 > gpurun_out/s5_ncu_bench.log 2>&1
fi
bash scripts/ncu_pass.sh config4 s5_sor_c4_red
tail -1 gpurun_out/s5_sor_c4_red.log
ls -la gpurun_out | tail -20
