# per-sweep time of library variants (variants/NAME.so) on configs 1 and 2 (default kernel)
mkdir -p gpurun_out
for v in "$@"; do
  for c in config1 config2; do
    SUBSURF_B200_LIB=variants/$v.so timeout 300 python scripts/sweep_rate.py $c > gpurun_out/rv_${v}_$c.json 2> gpurun_out/rv_${v}_$c.err
  done
done
