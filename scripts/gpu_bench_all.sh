# bench lines of configs 1, 2, 4, 0 + the reference arm, the launch list and steady-state
# ncu captures of a red pass on configs 1, 2 and 4 (gpurun_out/)
mkdir -p gpurun_out
timeout 300 python bench.py > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 300 python bench.py --config config2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --config config4 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 300 python bench.py --config config0 > gpurun_out/bench_c0.json 2> gpurun_out/bench_c0.err
[ -n "$REF" ] && timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
[ -n "$LAUNCHES" ] && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
[ -n "$NCU" ] && for c in $NCU; do timeout 600 scripts/ncu_pass.sh $c ${c}_red_s5; done
true
