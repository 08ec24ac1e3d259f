mkdir -p gpurun_out
for c in config1 config2; do
timeout 120 python scripts/sweep_rate.py $c | sed "s/^/h1M /"
for v in h0 h1k h20k; do SUBSURF_B200_LIB=variants/$v.so timeout 120 python scripts/sweep_rate.py $c | sed "s/^/$v /"; done
timeout 120 python scripts/sweep_rate.py $c | sed "s/^/h1M /"
done
