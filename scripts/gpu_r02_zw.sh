#!/bin/bash
# session-3 evidence: smoke, GPU suite, bench lines (config 4 default, configs 1 and 2), the
# reference arm on config 4, the launch list of exactly two timed config-4 steps
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_w3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests_w3.log
tail -2 gpurun_out/gpu_tests_w3.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4_w3.json 2> gpurun_out/bench_c4_w3.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4_w3.json')); print('c4', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline'].get('assemble_ms_per_step'), d['clocks'])"
timeout 900 python bench.py --config config1 --steps 20 --warmup 3 > gpurun_out/bench_c1_w3.json 2> gpurun_out/bench_c1_w3.err
python -c "import json; d=json.load(open('gpurun_out/bench_c1_w3.json')); print('c1', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 python bench.py --config config2 --steps 5 --warmup 3 > gpurun_out/bench_c2_w3.json 2> gpurun_out/bench_c2_w3.err
python -c "import json; d=json.load(open('gpurun_out/bench_c2_w3.json')); print('c2', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 1200 python bench.py --impl reference --steps 4 --warmup 3 > gpurun_out/bench_ref_c4_w3.json 2> gpurun_out/bench_ref_c4_w3.err
python -c "import json; d=json.load(open('gpurun_out/bench_ref_c4_w3.json')); print('ref', d.get('value'), d.get('ms_per_step'), d.get('cpu_baseline',{}).get('cores'))"
if timeout 600 python scripts/step_launch_list.py config4 2 > gpurun_out/sll_w3.log 2>&1; then
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches_step_c4_w3.csv python scripts/step_launch_list.py config4 2 > gpurun_out/ncu_sll_w3.log 2>&1
fi
ls -la gpurun_out/launches_step_c4_w3.csv
