mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_slabs.py -x -q -k "kwave" > gpurun_out/kw_tests.log 2>&1; echo "rc=$?" >> gpurun_out/kw_tests.log
for k in tma kwave; do SUBSURF_KERNEL=$k timeout 120 python scripts/sweep_rate.py config1 > gpurun_out/kw_rate_$k.json 2> gpurun_out/kw_rate_$k.err; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sor_kwave -s 5 -c 1 -o gpurun_out/kw_c1 -f env SUBSURF_KERNEL=kwave python scripts/sweep_rate.py config1 > gpurun_out/kw_ncu.log 2>&1
