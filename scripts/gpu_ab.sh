# A/B: per-sweep time of library variants (variants/NAME.so) on configs 1 and 2,
# then one ncu --set full capture of a steady-state red pass per variant (config 1).
mkdir -p gpurun_out
for v in "$@"; do
  for c in config1 config2; do
    SUBSURF_B200_LIB=variants/$v.so timeout 300 python scripts/sweep_rate.py $c > gpurun_out/ab_${v}_$c.json 2> gpurun_out/ab_${v}_$c.err
  done
done
for v in "$@"; do
  SUBSURF_B200_LIB=variants/$v.so timeout 600 scripts/ncu_pass.sh config1 ab_${v}_c1
done
