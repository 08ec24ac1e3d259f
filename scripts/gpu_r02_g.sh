#!/bin/bash
# smoke, ncu launch list of the config-4 bench command, ncu --set full of a config-4 red pass
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_g.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_g.log
if timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g.json 2>&1; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
     --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
fi
timeout 900 bash scripts/ncu_pass.sh config4 c4_red_r02
tail -2 gpurun_out/smoke_g.log; ls -la gpurun_out/*.ncu-rep gpurun_out/launches_c4.csv
