#!/bin/bash
# final session-3 evidence with 32-plane items: bench configs 4 / 1 / 2, config-4 launch list, one
# steady-state red pass capture of config 4
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4_fin.json 2> gpurun_out/bench_c4_fin.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4_fin.json')); print('c4', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 python bench.py --config config1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1_fin.json 2> gpurun_out/bench_c1_fin.err
python -c "import json; d=json.load(open('gpurun_out/bench_c1_fin.json')); print('c1', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 python bench.py --config config2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_fin.json 2> gpurun_out/bench_c2_fin.err
python -c "import json; d=json.load(open('gpurun_out/bench_c2_fin.json')); print('c2', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
if timeout 600 python scripts/step_launch_list.py config4 2 > gpurun_out/sll_fin.log 2>&1; then
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches_step_c4_fin.csv python scripts/step_launch_list.py config4 2 > gpurun_out/ncu_sll_fin.log 2>&1
fi
bash scripts/ncu_pass.sh config4 sor_c4_red_fin
tail -1 gpurun_out/sor_c4_red_fin.log
