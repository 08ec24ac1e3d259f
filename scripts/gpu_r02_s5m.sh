#!/bin/bash
# session 5 final: whole GPU suite (-x, as the driver runs it), smoke, the default bench line and the
# reference arm, configs 1 / 2, one steady-state red pass capture
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/s5m_suite.log
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1 | tee gpurun_out/s5m_smoke.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/s5m_bench_c4.json 2> gpurun_out/s5m_bench_c4.err
python -c "import json; d=json.load(open('gpurun_out/s5m_bench_c4.json')); print('c4', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['cpu_baseline']['value'])"
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/s5m_bench_ref_c4.json 2> gpurun_out/s5m_bench_ref_c4.err
python -c "import json; d=json.load(open('gpurun_out/s5m_bench_ref_c4.json')); print('ref c4', d['value'], d['ms_per_step'], d['steps'])"
timeout 900 python bench.py --config config1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/s5m_bench_c1.json 2> gpurun_out/s5m_bench_c1.err
python -c "import json; d=json.load(open('gpurun_out/s5m_bench_c1.json')); print('c1', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
timeout 900 python bench.py --config config2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5m_bench_c2.json 2> gpurun_out/s5m_bench_c2.err
python -c "import json; d=json.load(open('gpurun_out/s5m_bench_c2.json')); print('c2', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
