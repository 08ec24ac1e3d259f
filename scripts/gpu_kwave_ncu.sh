mkdir -p gpurun_out
SUBSURF_KERNEL=kwave timeout 300 ncu --set full --clock-control none --import-source on -k regex:sor_kwave -s 5 -c 1 -o gpurun_out/kw_c1 -f python scripts/sweep_rate.py config1 > gpurun_out/kw_ncu.log 2>&1
